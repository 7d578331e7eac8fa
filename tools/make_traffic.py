"""profiles/traffic.json from the ncu --set full captures of tools/gpu_round.sh:
per workload the dominant kernel's dram__bytes_read.sum + dram__bytes_write.sum
for one launch (bench.py reports it as roofline.traffic), and a text summary of
each capture under profiles/ (prefix = argv[1], e.g. r01)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    names, units, vals = rows[0], rows[1], rows[2]
    return {n: (v, u) for n, u, v in zip(names, units, vals)}


def main():
    prefix = sys.argv[1] if len(sys.argv) > 1 else "r02"
    outdir = os.environ.get("TRAFFIC_OUT", os.path.join(ROOT, "profiles"))  # on the GPU box: under gpurun_out/
    os.makedirs(outdir, exist_ok=True)
    path = os.path.join(outdir, "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for w in ["c2", "c2a", "c1", "c3", "c4", "c4adj", "c5", "rm"]:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{w}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m = raw(rep)
        tot = 0.0
        for key in ["dram__bytes_read.sum", "dram__bytes_write.sum"]:
            v, u = m[key]
            tot += float(v.replace(",", "")) * UNITS.get(u, 1)
        t, tu = m["gpu__time_duration.sum"]
        data[w] = {"bytes": int(tot), "kernel": m.get("Kernel Name", ("?", ""))[0][:120],
                   "ncu_time_us": float(t.replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
                                                                  "msecond": 1e3, "ms": 1e3}.get(tu, 1),
                   "source": f"ncu --set full --clock-control none, one launch ({prefix})"}
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                              capture_output=True, text=True).stdout
        with open(os.path.join(outdir, f"{prefix}_ncu_{w}.txt"), "w") as f:
            f.write(summ)
    with open(path, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
