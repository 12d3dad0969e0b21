"""What a 20-step timed burst of the c4 R(U) apply measures under the
bench's conditions: after a long warm loop or a 0.1 s pre-roll, with and
without the NVML clock-sampler thread.  Prints one JSON object."""
import json
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
U = [torch.as_tensor(C.random_slab(cfg), device="cuda").clone() for _ in range(3)]
un = [torch.as_tensor(C.initial_state(cfg), device="cuda").clone() for _ in range(3)]
R = [torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda") for _ in range(3)]


def step(i):
    op.st_residual(0.0, cfg.dt, un[i % 3], U[i % 3], out=R[i % 3])


def burst(K=20, gate=1_800_000):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    torch.cuda._sleep(gate)
    e0.record()
    for i in range(K):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / K


def sampler(stop):
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        N.nvmlDeviceGetCurrentClocksEventReasons(h)
        stop.wait(0.005)
    N.nvmlShutdown()


out = {}
for i in range(2000):
    step(i)
out["warm_K20"] = [burst() for _ in range(5)]
out["warm_K200"] = [burst(200, 18_000_000) for _ in range(3)]
t0 = time.perf_counter()
i = 0
while time.perf_counter() - t0 < 0.1:
    for _ in range(200):
        step(i)
        i += 1
    torch.cuda.synchronize()
out["after_preroll_K20"] = [burst() for _ in range(5)]
stop = threading.Event()
th = threading.Thread(target=sampler, args=(stop,), daemon=True)
th.start()
time.sleep(0.05)
out["with_sampler_K20"] = [burst() for _ in range(5)]
stop.set()
th.join()
out["after_sampler_K20"] = [burst() for _ in range(5)]
# R(U) one launch per 3 buffers vs the same buffer
def burst_same(K=20):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    torch.cuda._sleep(1_800_000)
    e0.record()
    for i in range(K):
        op.st_residual(0.0, cfg.dt, un[0], U[0], out=R[0])
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / K
out["same_buffers_K20"] = [burst_same() for _ in range(3)]
print(json.dumps(out))
