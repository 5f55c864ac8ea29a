"""Where the packed end-to-end step goes: upload, decode, refresh, BFS,
widen + read-back, each timed alone (CUDA events), s24."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200 import _native  # noqa: E402
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.io import pack_csr_device  # noqa: E402
from paper_1701_01170_b200.primitives.bfs import bfs_device  # noqa: E402

dg = rmat_device_graph(24, 16, 0)
packed = pack_csr_device(dg)
print("packed bytes", packed.nbytes)


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
        wall = (time.perf_counter() - t0) * 1e3
    print(f"{name:10s} {best:8.3f} ms (wall {wall:.3f})")


timed("upload", lambda: dg.upload_packed_(packed))
rc, rd, rb, cc, cd, cb = dg._pack_stage[0]
timed("dec_rows", lambda: _native.call("gfx_csr_unpack", dg.ctx.handle, _native.ptr(rc),
                                       _native.ptr(rd), _native.ptr(rb), dg.num_vertices + 1,
                                       _native.ptr(dg.row), 8, 0))
timed("dec_cols", lambda: _native.call("gfx_csr_unpack", dg.ctx.handle, _native.ptr(cc),
                                       _native.ptr(cd), _native.ptr(cb), dg.num_edges,
                                       _native.ptr(dg.col), 4, 0))
timed("refresh", lambda: _native.call("gfx_graph_refresh", dg.handle))
timed("bfs", lambda: bfs_device(dg, 0, direction="auto"))
h = [t.numel() for t in packed.row + packed.col]
print("stream sizes", h, [t.is_pinned() for t in packed.row + packed.col])

up = pack_csr_device(dg, upper=True)
print("upper packed bytes", up.nbytes)
timed("upload_up", lambda: dg.upload_packed_(up))
timed("decode_up", lambda: dg.decode_packed_())
timed("rebuild", lambda: _native.call("gfx_graph_rebuild_upper", dg.handle,
                                      _native.ptr(dg._upper_tmp[0]), _native.ptr(dg._upper_tmp[1]),
                                      dg.num_edges // 2))
