"""One gfx_graph_rebuild_upper at s24 after a warm-up (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200 import _native  # noqa: E402
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.io import pack_csr_device  # noqa: E402

dg = rmat_device_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, 0)
up = pack_csr_device(dg, upper=True)
dg.upload_packed_(up)
dg.decode_packed_()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
_native.call("gfx_graph_rebuild_upper", dg.handle, _native.ptr(dg._upper_tmp[0]),
             _native.ptr(dg._upper_tmp[1]), dg.num_edges // 2)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
