"""DRAM bandwidth probes on the box: write-only (fill), read+write 1:1 (copy), and a 1:3 read:write mix."""
import torch
n = 2_424_000_000 // 8
a = torch.empty(n, dtype=torch.int64, device="cuda")
b = torch.empty(n, dtype=torch.int64, device="cuda")
c = torch.empty(3 * n, dtype=torch.int64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


ms = t(lambda: a.fill_(7))
print(f"fill   {n * 8 / 1e9:.2f} GB written: {ms:.3f} ms -> {n * 8 / ms / 1e6:.0f} GB/s")
ms = t(lambda: b.copy_(a))
print(f"copy   {2 * n * 8 / 1e9:.2f} GB moved:   {ms:.3f} ms -> {2 * n * 8 / ms / 1e6:.0f} GB/s")
v = c.view(3, n)
ms = t(lambda: torch.add(a.unsqueeze(0), v, out=v))
print(f"1r3w+3r (a + c -> c, c 3x larger): {ms:.3f} ms -> {7 * n * 8 / ms / 1e6:.0f} GB/s")
ms = t(lambda: v.copy_(a.unsqueeze(0).expand(3, n)))
print(f"1 read : 3 writes (broadcast copy): {ms:.3f} ms -> {4 * n * 8 / ms / 1e6:.0f} GB/s")
