"""Dependent-load latency on this GPU (one thread, pointer chase): an L2-sized
span vs spans far beyond L2 / TLB reach, at line (128 B) stride."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_01170_b200 import _native  # noqa: E402

ctx = _native.Context(0)
g = torch.Generator(device="cpu").manual_seed(0)
for span_mb in (1, 2, 16, 64, 256, 1024, 4096):
    words = span_mb * (1 << 20) // 4
    lines = words // 32
    perm = torch.randperm(lines, generator=g)
    nxt = torch.empty(lines, dtype=torch.int64)
    nxt[perm] = torch.roll(perm, -1)  # cycle through lines in random order
    buf = torch.zeros(words, dtype=torch.int32)
    buf[torch.arange(lines) * 32] = (nxt * 32).to(torch.int32)
    bd = buf.cuda()
    cyc = ctypes.c_double()
    _native.call("gfx_debug_chase", ctx.handle, ctypes.c_void_p(bd.data_ptr()), 20000, 0,
                 ctypes.byref(cyc))
    print(f"span {span_mb:5d} MB  {cyc.value:8.1f} cycles/load")
    del bd
