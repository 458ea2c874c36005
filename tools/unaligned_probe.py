"""K3 on an unaligned geometry (rows not 16-byte multiples): 8 x 2046x1536,
30 frames, given maps; ms per call and GB/s on 6 B/px."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib

N, H, W, K, B = 8, 1536, 2046, 16, 30
src = torch.randint(0, 256, (B, N, H, W, 3), dtype=torch.uint8, device="cuda")
out = torch.empty_like(src)
g = torch.full((B, N - 1, 2, K, 3), 1.2, dtype=torch.float64, device="cuda")
o = torch.full_like(g, 3.0)
call = lambda: _lib.call("camx_apply_array", src.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W,
                         K, g.data_ptr(), o.data_ptr(), None)
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"unaligned K3 (W={W}): {ms:.3f} ms = {6 * src.numel() / 3 / ms / 1e6:.0f} GB/s")
