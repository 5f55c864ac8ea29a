"""One expansion of the s24 BFS level-2 frontier with a chosen functor variant
(for ncu captures): python tools/expand_prof.py <variant> [scale]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200.generators import rmat_device_graph

    variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    level = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    dg = rmat_device_graph(scale, 16, 0)
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    full, _, _ = bfs_device(dg, 0, direction="push")
    F = torch.nonzero(full == level - 1).flatten().to(torch.int32)
    labels = full.clone()
    labels[labels >= level] = _native.UNVISITED32
    ms, cnt = ctypes.c_float(), ctypes.c_int64()
    for _ in range(2):
        lab = labels.clone()
        torch.cuda.synchronize()
        _native.call("gfx_debug_expand", dg.handle, _native.ptr(F), F.numel(), variant,
                     _native.ptr(lab), level, ctypes.byref(ms), ctypes.byref(cnt))
    print("variant", variant, "ms", ms.value, "emitted", cnt.value)


if __name__ == "__main__":
    main()
