"""Pinned host<->device copy bandwidth on this box (one direction, then both at once)."""
import torch, time
n = 1 << 28  # 2 GiB of float64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, f in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); f(); e.record(); torch.cuda.synchronize()
    print(name, round(n * 8 / s.elapsed_time(e) / 1e6, 1), "GB/s")
# concurrent both directions
st1, st2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True); d2 = torch.empty_like(d)
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(st1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(st2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("bidir each", round(n * 8 / dt / 1e9, 1), "GB/s")
