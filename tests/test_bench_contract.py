"""bench.py contract checks that run on CPU: the reference arm's workload
table equals the product's configs, both arms emit the same `config`, and
the reference arm runs the oracle alone (no product module, no
libstg_cuda.so mapped)."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2201_05800_b200 import configs as C  # noqa: E402


@pytest.mark.parametrize("name", sorted(bench.REF_WORKLOADS))
def test_reference_workloads_match_configs(name):
    w, cfg = bench.REF_WORKLOADS[name], C.CONFIGS[name]
    for k in ("dim", "degree", "n_tau", "cells", "lower", "upper", "velocity", "dt", "seed"):
        assert tuple(np.atleast_1d(w[k])) == tuple(np.atleast_1d(getattr(cfg, k))), k
    assert bench.workload_sizes(w) == (cfg.n_sdof, cfg.n_dof)


def test_reference_inputs_bitwise_equal_product_inputs():
    import oracle as O
    pr, U, un = bench.oracle_inputs("c4", O)
    cfg = C.CONFIGS["c4"]
    assert np.array_equal(U, C.random_slab(cfg))
    assert np.array_equal(un, C.initial_state(cfg))


def test_reference_arm_loads_only_the_oracle():
    code = (
        "import sys, json, io, contextlib; sys.argv=['bench.py','--impl','reference','--steps','2',"
        "'--warmup','3','--workload','c4']; sys.path.insert(0, %r); import bench;"
        "buf=io.StringIO();\n"
        "with contextlib.redirect_stdout(buf): bench.main()\n"
        "maps=open('/proc/self/maps').read();"
        "print(json.dumps({'line': json.loads(buf.getvalue().strip().splitlines()[-1]),"
        "'product_imported': any(m.startswith('paper_2201_05800_b200') for m in sys.modules),"
        "'stg_mapped': 'libstg_cuda.so' in maps, 'oracle_mapped': 'liboracle' in maps}))"
    ) % str(ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert not out["product_imported"] and not out["stg_mapped"] and out["oracle_mapped"]
    line = out["line"]
    assert line["impl"] == "reference" and line["warmup"] == 3 and line["steps"] == 2
    assert line["config"] == bench.bench_config("c4", 1)
    assert line["cpu_baseline"]["cores"] >= 1 and line["e2e"]["h2d_bytes_per_step"] == 0
