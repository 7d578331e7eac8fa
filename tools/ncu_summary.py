"""Compact text summary of an ncu --set full report (one kernel): time, DRAM
bytes, throughput, occupancy, stall breakdown, instruction mix.
Usage: python tools/ncu_summary.py rep.ncu-rep [title] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
u = dict(zip(h, units))


def g(k):
    x = d.get(k, "")
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return x


print(f"# ncu --set full summary: {title}")
print(f"kernel: {d.get('Kernel Name', '?')[:160]}")
print(f"grid {d.get('launch__grid_size')} x block {d.get('launch__block_size')}, regs/thread {d.get('launch__registers_per_thread')}, "
      f"dyn smem/block {d.get('launch__shared_mem_per_block_dynamic')} {u.get('launch__shared_mem_per_block_dynamic')}")
dur = g("gpu__time_duration.sum")
print(f"gpu__time_duration.sum = {dur} {u.get('gpu__time_duration.sum')}")
rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
print(f"dram__bytes_read.sum = {rd} {u.get('dram__bytes_read.sum')}; dram__bytes_write.sum = {wr} {u.get('dram__bytes_write.sum')}")
for k in ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
          "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
          "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "launch__occupancy_limit_shared_mem",
          "launch__occupancy_limit_registers"]:
    if k in d:
        print(f"{k} = {d[k]} {u.get(k, '')}")
st = {}
for k, x in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(x.replace(",", ""))
        except ValueError:
            pass
t = sum(st.values()) or 1
print("warp stall samples (top):")
for k, x in sorted(st.items(), key=lambda z: -z[1])[:10]:
    print(f"  {k:28s} {100 * x / t:5.1f}%")
