"""Raw pinned-memory PCIe bandwidth: H2D, D2H, and both at once (1 GiB)."""
import torch
n = 1 << 27  # 1 GiB of float64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)


ms = t(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D {8 * n / ms / 1e6:.1f} GB/s")
ms = t(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H {8 * n / ms / 1e6:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


ms = t(both)
print(f"both directions at once: {8 * n / ms / 1e6:.1f} GB/s each")
