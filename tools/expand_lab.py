"""Break the push expansion of the s24 BFS levels into stream / probe / claim
costs (gfx_debug_expand).  GPU only."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    dg = rmat_device_graph(scale, 16, 0)
    labels, _, st = bfs_device(dg, 0, direction="push")
    deg = dg.row[1:] - dg.row[:-1]
    for depth in (2, 3):
        F = torch.nonzero(labels == depth - 1).flatten().to(torch.int32)
        slots = int(deg[F.long()].sum().item())
        base = labels.clone()
        base[base >= depth] = _native.UNVISITED32
        for variant, name in ((0, "strm16"), (3, "strm8"), (1, "probe"), (2, "claim")):
            times = []
            for _ in range(4):
                lab = base.clone()
                torch.cuda.synchronize()
                ms = ctypes.c_float()
                cnt = ctypes.c_int64()
                _native.call("gfx_debug_expand", dg.handle, _native.ptr(F), F.numel(), variant,
                             _native.ptr(lab), depth, ctypes.byref(ms), ctypes.byref(cnt))
                times.append(ms.value)
            t = min(times[1:])
            print(f"level {depth} |F|={F.numel():>9} slots={slots:>11} {name:<6} {t:8.3f} ms "
                  f"{slots / t / 1e6:8.1f} Gslot/s  {4 * slots / t / 1e6:7.1f} GB/s(col)  "
                  f"emitted={cnt.value}")


if __name__ == "__main__":
    main()
