"""What does plain HBM traffic of the c4 R(U) shape cost on this B200?
read 64 MiB (+16 MiB) and write 64 MiB with rotation (no L2 reuse)."""
import json
import torch

n_dof, n_sdof = 8388608, 2097152
sets = 3
U = [torch.rand(n_dof, dtype=torch.float64, device="cuda") for _ in range(sets)]
R = [torch.empty(n_dof, dtype=torch.float64, device="cuda") for _ in range(sets)]
w = [torch.rand(n_sdof, dtype=torch.float64, device="cuda") for _ in range(sets)]
s = torch.cuda.current_stream()


def bench(fn, reps=400):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(s)
    for i in range(reps):
        fn(i)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


out = {}
t = bench(lambda i: R[i % sets].copy_(U[i % sets]))
out["copy_64MiB_us"] = t
out["copy_GBps"] = 2 * 8 * n_dof / t / 1e3
t = bench(lambda i: torch.mul(U[i % sets], 2.0, out=R[i % sets]))
out["scale_us"] = t
big = torch.rand(1 << 28, dtype=torch.float64, device="cuda")
big2 = torch.empty_like(big)
t = bench(lambda i: big2.copy_(big), reps=20)
out["copy_2GiB_GBps"] = 2 * 8 * (1 << 28) / t / 1e3
print(json.dumps(out))
