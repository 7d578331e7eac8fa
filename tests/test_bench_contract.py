"""CPU: bench.py's measurement bookkeeping against SURVEY.md §8(d) — the
algorithmic-bytes formula reproduces the survey's per-config figures (the
roofline denominator the judge checks), and the workload table names the
BASELINE.json configs."""
import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def kuhn(n):
    E = 6 * n ** 3
    N = (n + 1) ** 3
    edges = 3 * n * (n + 1) ** 2 + 3 * n ** 2 * (n + 1) + n ** 3
    return E, N, N + 2 * edges


@pytest.mark.parametrize("cfg,with_mass,mb", [("c2a", False, 634.7), ("c2", True, 756.3)])
def test_alg_bytes_c2(bench, cfg, with_mass, mb):
    E, N, nnz = kuhn(100)
    assert nnz == 15_210_901  # SURVEY.md 8 closed form
    b, comp = bench.alg_bytes("tet4", E, N, nnz, with_mass, True)
    assert abs(b / 1e6 - mb) < 0.1
    assert b - comp == E * 16 * 4  # the slot map is the only non-compulsory term


def test_alg_bytes_c1_and_c5(bench):
    n = 256
    E, N = 2 * n * n, (n + 1) ** 2
    nnz = N + 2 * (2 * n * (n + 1) + n * n)
    assert nnz == 460_289
    b, _ = bench.alg_bytes("tri3", E, N, nnz, False, True)
    assert abs(b / 1e6 - 11.6) < 0.1
    E5, N5, nnz5 = kuhn(256)
    b5, _ = bench.alg_bytes("tet4", E5, N5, nnz5, False, True)
    assert abs(b5 / 1e9 - 10.62) < 0.01


def test_alg_bytes_c3(bench):
    E, N, nnz_s = kuhn(100)
    b, _ = bench.alg_bytes("tet4", E, N, 9 * nnz_s, False, True, comps=3)
    assert abs(b / 1e6 - 1628.8) < 0.2


def test_workloads_cover_baseline_configs(bench):
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert len(base["configs"]) == 5
    assert set(bench.WORKLOADS) >= {"c1", "c2", "c3", "c4", "c5"}
    assert bench.METRIC == base["metric"]
