"""Host<->device copy rates of this box (pinned memory, 1 GiB): H2D alone, D2H alone, both at
once on two streams.  The e2e bench line cannot beat the concurrent figure."""
import torch

n = 1 << 27  # 1 GiB of fp64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 8 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D {t:.2f} ms  {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H {t:.2f} ms  {gb / t * 1e3:.1f} GB/s")
t = timed(both)
print(f"H2D+D2H concurrent {t:.2f} ms  {2 * gb / t * 1e3:.1f} GB/s total")
