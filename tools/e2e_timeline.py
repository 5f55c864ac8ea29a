"""Timeline of the double-buffered packed e2e loop (bench.e2e): per step the
upload (upload stream) and decode / BFS / read-back (compute and read-back
streams) start and end times from CUDA events, s24; plus uploads alone."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.io import pack_csr_device  # noqa: E402
from paper_1701_01170_b200.primitives.bfs import bfs_device  # noqa: E402

dg = rmat_device_graph(24, 16, 0)
packed = pack_csr_device(dg, upper=len(sys.argv) > 1 and sys.argv[1] == "upper")
n = dg.num_vertices
comp = torch.cuda.current_stream()
up, dn = torch.cuda.Stream(), torch.cuda.Stream()
labels = torch.empty(n, dtype=torch.int32, device="cuda")
preds = torch.empty(n, dtype=torch.int32, device="cuda")
wide = torch.empty(2 * n, dtype=torch.int64, device="cuda")
host = torch.empty(2 * n, dtype=torch.int64, pin_memory=True)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


for rep in range(3):
    torch.cuda.synchronize()
    t0 = ev(comp)
    marks = []
    for k in range(5):
        with torch.cuda.stream(up):
            up.wait_stream(comp) if k == 0 else None
            a = ev(up)
            dg.upload_packed_(packed, slot=0)
            b = ev(up)
        marks.append(("upload", a, b))
    torch.cuda.synchronize()
    print("uploads alone:", [round(a.elapsed_time(b), 2) for _, a, b in marks])

for rep in range(6):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t0 = ev(comp)
    marks = []
    host_t = []
    up.wait_stream(comp)
    with torch.cuda.stream(up):
        a = ev(up); dg.upload_packed_(packed, slot=0); b = ev(up)
    marks.append(("up0", a, b))
    up_ev = [b, None]
    dec_ev = [None, None]
    for k in range(5):
        s = k % 2
        if k + 1 < 5:
            with torch.cuda.stream(up):
                if dec_ev[1 - s] is not None:
                    up.wait_event(dec_ev[1 - s])
                a = ev(up); dg.upload_packed_(packed, slot=1 - s); b = ev(up)
            marks.append((f"up{k+1}", a, b))
            up_ev[1 - s] = b
        comp.wait_event(up_ev[s])
        a = ev(comp)
        h0 = time.perf_counter()
        dg.decode_packed_(slot=s)
        h1 = time.perf_counter()
        dec_ev[s] = ev(comp)
        bfs_device(dg, 0, direction="auto", labels=labels, preds=preds)
        h2 = time.perf_counter()
        host_t.append((k, round((h0 - w0) * 1e3, 2), round((h1 - h0) * 1e3, 2), round((h2 - h1) * 1e3, 2)))
        wide[:n].copy_(labels)
        wide[n:].copy_(preds)
        b = ev(comp)
        marks.append((f"dec+bfs{k}", a, b))
        with torch.cuda.stream(dn):
            dn.wait_event(b)
            a2 = ev(dn); host.copy_(wide, non_blocking=True); b2 = ev(dn)
        marks.append((f"d2h{k}", a2, b2))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) * 1e3
    print(f"rep {rep}: wall {wall:.1f} ms = {wall/5:.2f} per step")
    print("   host (step, decode call at, decode call ms, bfs call ms):", host_t)
    for name, a, b in marks:
        print(f"   {name:10s} {t0.elapsed_time(a):8.2f} -> {t0.elapsed_time(b):8.2f}  ({a.elapsed_time(b):.2f})")
