"""Real-rank device-resident partitioned BFS with P processes on ONE GPU
(CUDA IPC within the device, gloo for the handle exchange): the kernels of
the two processes meet at device flag barriers.  Compares the gathered
labels with the single-GPU BFS.   python tools/pd_two_proc.py [scale] [P]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(r, P, scale, port, out, prim):
    import torch
    import torch.distributed as tdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=r, world_size=P)
    torch.cuda.set_device(0)
    from paper_1701_01170_b200.dist import DeviceResidentRank, DeviceResidentSsspRank
    from paper_1701_01170_b200.generators import rmat_device_graph

    if prim == "sssp":
        dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
        eng = DeviceResidentSsspRank(dg, P, r)
        tdist.barrier()
        lab, prd, st = eng.run(0, 32)
        out[r] = (lab.cpu().numpy().tolist(), [st.iterations], st.device_ms)
    else:
        dg = rmat_device_graph(scale, 16, 0)
        eng = DeviceResidentRank(dg, P, r)
        tdist.barrier()
        lab, prd, st, levels = eng.run(0, direction="auto")
        out[r] = (lab.cpu().numpy().tolist(), [lv["mode"] for lv in levels], st.device_ms)
    tdist.barrier()
    eng.close()
    tdist.destroy_process_group()


if __name__ == "__main__":
    import multiprocessing as mp

    import numpy as np
    import torch

    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    prim = sys.argv[3] if len(sys.argv) > 3 else "bfs"
    mp.set_start_method("spawn")
    mgr = mp.Manager()
    out = mgr.dict()
    procs = [mp.Process(target=worker, args=(r, P, scale, 29611 + P, out, prim)) for r in range(P)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    if any(p.is_alive() for p in procs):
        for p in procs:
            p.kill()
        print("TIMEOUT")
        sys.exit(2)
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    if prim == "sssp":
        dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
        want = sssp_device(dg, 0, delta=32)[0].cpu().numpy()
    else:
        dg = rmat_device_graph(scale, 16, 0)
        want = bfs_device(dg, 0, direction="auto")[0].cpu().numpy()
    got = np.empty_like(want)
    for r in range(P):
        got[r::P] = np.array(out[r][0], dtype=want.dtype)
    print(f"{prim} P={P} s{scale} labels equal:", bool(np.array_equal(got, want)), "trace", out[0][1], "ms",
          [round(out[r][2], 3) for r in range(P)])
