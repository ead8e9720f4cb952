"""Practical HBM read-bandwidth ceiling on this box: torch reductions over
>L2 buffers (reference point for the weight-streaming GEMV)."""
import torch
x = torch.empty(4 * 235 * 2**20 // 2, dtype=torch.bfloat16, device="cuda").normal_()
ys = [torch.empty_like(x).normal_() for _ in range(3)]
for name, fn in [("sum_bf16", lambda t: t.sum()), ("amax", lambda t: t.abs().amax()),
                 ("view_f32_sum", lambda t: t.view(torch.float32).sum())]:
    bufs = [x] + ys
    for b in bufs:
        fn(b)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 12
    for i in range(n):
        fn(bufs[i % 4])
    e.record()
    e.synchronize()
    dt = a.elapsed_time(e) / 1e3 / n
    print(f"{name}: {x.numel() * 2 / dt / 1e9:.0f} GB/s read ({dt * 1e6:.1f} us)")
