"""PCIe schedule probe for the host-buffer R(U) call (c4 bytes: U + u_n in,
R out, pinned).  Times copy-only schedules against the real pipelined call
so the gap between the call and its transfer bound can be attributed:

  h2d_1s / h2d_2s        80 MiB in, one stream vs split over two streams
  duplex_1s / duplex_2s  80 MiB in + 64 MiB out at once (in on 1 or 2 streams)
  chain_K                the call's chunk schedule with copies only (chunk k's
                         D2H waits on chunk k's H2D), K = 4, 8, 16
  call                   stg_st_residual_host itself

Prints one JSON object (ms per call, CUDA events, best of 5 rounds)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
nd, ns = cfg.n_dof, cfg.n_sdof
hU = torch.empty(nd, dtype=torch.float64, pin_memory=True)
hu = torch.empty(ns, dtype=torch.float64, pin_memory=True)
hR = torch.empty(nd, dtype=torch.float64, pin_memory=True)
dU = torch.empty(nd, dtype=torch.float64, device="cuda")
du = torch.empty(ns, dtype=torch.float64, device="cuda")
dR = torch.empty(nd, dtype=torch.float64, device="cuda")
main = torch.cuda.current_stream()
S = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(main)
        for _ in range(reps):
            fn()
        e1.record(main)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def fork(*ss):
    for s in ss:
        s.wait_stream(main)


def join(*ss):
    for s in ss:
        main.wait_stream(s)


def h2d_1s():
    dU.copy_(hU, non_blocking=True)
    du.copy_(hu, non_blocking=True)


def h2d_2s():
    fork(S[0], S[1])
    h = nd // 2
    with torch.cuda.stream(S[0]):
        dU[:h].copy_(hU[:h], non_blocking=True)
    with torch.cuda.stream(S[1]):
        dU[h:].copy_(hU[h:], non_blocking=True)
        du.copy_(hu, non_blocking=True)
    join(S[0], S[1])


def duplex(two):
    def f():
        fork(S[0], S[1], S[2])
        if two:
            h = nd // 2
            with torch.cuda.stream(S[0]):
                dU[:h].copy_(hU[:h], non_blocking=True)
            with torch.cuda.stream(S[1]):
                dU[h:].copy_(hU[h:], non_blocking=True)
                du.copy_(hu, non_blocking=True)
        else:
            with torch.cuda.stream(S[0]):
                dU.copy_(hU, non_blocking=True)
                du.copy_(hu, non_blocking=True)
        with torch.cuda.stream(S[2]):
            hR.copy_(dR, non_blocking=True)
        join(S[0], S[1], S[2])
    return f


def chain(K):
    # chunk k of each temporal block: U[t*ns + a : t*ns + b], u_n[a:b]
    nt = cfg.n_tau
    bounds = [ns * k // K for k in range(K + 1)]
    Uv, Rv = dU.view(nt, ns), dR.view(nt, ns)
    hUv, hRv = hU.view(nt, ns), hR.view(nt, ns)

    def f():
        fork(S[0], S[2])
        evs = []
        for k in range(K):
            a, b = bounds[k], bounds[k + 1]
            with torch.cuda.stream(S[0]):
                for t in range(nt):
                    Uv[t, a:b].copy_(hUv[t, a:b], non_blocking=True)
                du[a:b].copy_(hu[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(S[0])
                evs.append(e)
        for k in range(K):
            a, b = bounds[k], bounds[k + 1]
            S[2].wait_event(evs[k])
            with torch.cuda.stream(S[2]):
                for t in range(nt):
                    hRv[t, a:b].copy_(Rv[t, a:b], non_blocking=True)
        join(S[0], S[2])
    return f


out = {
    "h2d_1s": timed(h2d_1s), "h2d_2s": timed(h2d_2s),
    "d2h": timed(lambda: hR.copy_(dR, non_blocking=True)),
    "duplex_1s": timed(duplex(False)), "duplex_2s": timed(duplex(True)),
}
for K in (4, 8, 16):
    out[f"chain_{K}"] = timed(chain(K))
op = SlabOperator(**cfg.kwargs())
a, b, c = hu.numpy(), hU.numpy(), hR.numpy()
b[:] = C.random_slab(cfg)
a[:] = C.initial_state(cfg)
out["call"] = timed(lambda: op.st_residual_host(0.0, cfg.dt, a, b, out=c), reps=20)
print(json.dumps({k: round(v, 4) for k, v in out.items()}))
