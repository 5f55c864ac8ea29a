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
    dg = rmat_device_graph(scale, 16, 0)
    deg0 = int((dg.row[1] - dg.row[0]).item())
    F = dg.col[:deg0].clone()  # level-2 frontier = N(0)
    labels = torch.full((dg.num_vertices,), _native.UNVISITED32, dtype=torch.int32, device="cuda")
    labels[0] = 0
    labels[F.long()] = 1
    ms, cnt = ctypes.c_float(), ctypes.c_int64()
    for _ in range(2):
        lab = labels.clone()
        torch.cuda.synchronize()
        _native.call("gfx_debug_expand", dg.handle, _native.ptr(F), F.numel(), variant,
                     _native.ptr(lab), 2, ctypes.byref(ms), ctypes.byref(cnt))
    print("variant", variant, "ms", ms.value, "emitted", cnt.value)


if __name__ == "__main__":
    main()
