"""Is a camx launch on stream handle 0 (torch's default stream) ordered with
torch's own work on that stream?  A long K3 launch writes `out`; torch then
reads it on the current (default) stream without any other sync."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_03517_b200 import _lib  # noqa: E402

N, H, W, K, B = 8, 1536, 2048, 16, 30
src = torch.randint(0, 256, (B, N, H, W, 3), dtype=torch.uint8, device="cuda")
g = torch.full((B, N - 1, 2, K, 3), 1.5, dtype=torch.float64, device="cuda")
o = torch.zeros_like(g)
bad = 0
for it in range(20):
    out = torch.zeros_like(src)
    torch.cuda.synchronize()
    s0 = torch.cuda.current_stream()
    _lib.call("camx_apply_array", src.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K,
              g.data_ptr(), o.data_ptr(), s0.cuda_stream)
    # a torch kernel on the same (default) stream, right behind the launch
    last = out[-1, -1, -1, -1].clone()
    torch.cuda.synchronize()
    want = out[-1, -1, -1, -1]
    bad += int(not torch.equal(last, want))
print("stream handle", torch.cuda.current_stream().cuda_stream, "unordered reads:", bad, "of 20")
s = torch.cuda.Stream()
bad = 0
with torch.cuda.stream(s):
    for it in range(20):
        out = torch.zeros_like(src)
        _lib.call("camx_apply_array", src.data_ptr(), out.data_ptr(), B, 0, N, N, 0, H, W, K,
                  g.data_ptr(), o.data_ptr(), s.cuda_stream)
        last = out[-1, -1, -1, -1].clone()
        s.synchronize()
        bad += int(not torch.equal(last, out[-1, -1, -1, -1]))
print("side stream: unordered reads:", bad, "of 20")
