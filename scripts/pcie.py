import json, torch
n_in, n_out = 10485760, 8388608  # doubles: U+u_n (84 MB), R (67 MB)
hi = torch.empty(n_in, dtype=torch.float64, pin_memory=True)
ho = torch.empty(n_out, dtype=torch.float64, pin_memory=True)
di = torch.empty(n_in, dtype=torch.float64, device="cuda")
do = torch.empty(n_out, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
h2d = t(lambda: di.copy_(hi, non_blocking=True))
d2h = t(lambda: ho.copy_(do, non_blocking=True))
def both():
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bi = t(both)
print(json.dumps({"h2d_ms": h2d, "h2d_GBps": n_in*8/h2d/1e6, "d2h_ms": d2h, "d2h_GBps": n_out*8/d2h/1e6,
                  "bidir_ms": bi, "sequential_sum_ms": h2d + d2h}))
