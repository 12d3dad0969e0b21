"""World-size-2 (gloo, CPU) test of the multi-GPU bench logic: every rank runs
an independent replica (the north star is one GPU; DESIGN.md "replicas
only"), the job time is the max over ranks, and the value aggregates all
replicas' work."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws, r, local = bench.dist_env()
    my_ms = 10.0 + 5.0 * rank  # rank 1 is the slow replica
    ms = bench.reduce_max(my_ms, dist, "cpu")
    val = bench.whole_job_value(ws, 8388608, 100, ms)
    q.put((r, ws, local, ms, val))
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[0] for o in out] == [0, 1]
    assert all(o[1] == 2 for o in out)
    assert all(o[3] == 15.0 for o in out)  # max over ranks
    assert out[0][4] == pytest.approx(2 * 8388608 * 100 / 0.015)


def test_reference_arm_json_shape(monkeypatch, capsys):
    """--impl reference prints the contract's keys (tiny budget, rank 0)."""
    sys.path.insert(0, str(ROOT))
    import bench
    monkeypatch.setenv("STG_REF_BUDGET_S", "0.01")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "1",
                                      "--warmup", "3", "--workload", "c4"])
    # shrink the workload so the CPU run stays fast
    from paper_2201_05800_b200 import configs as C
    small = C.CONFIGS["c4"].scaled((8, 8, 8))
    monkeypatch.setitem(C.CONFIGS, "c4", small)
    assert bench.main() == 0
    import json
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "cpu_baseline", "e2e", "config"):
        assert k in line
    assert line["impl"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port"
