"""Single-GPU driver for ncu captures: build the R-MAT graph on the GPU, warm
up, then run the requested primitive a fixed number of times.

    python tools/prof_run.py --prim bfs --direction push --scale 24 --runs 1
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prim", default="bfs")
    ap.add_argument("--direction", default="auto")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--runs", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--delta", type=float, default=32)
    ap.add_argument("--timing", action="store_true", help="per-iteration CUDA events")
    a = ap.parse_args()
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph

    weights = (1, 64) if a.prim == "sssp" else None
    dg = rmat_device_graph(a.scale, 16, 0, weights=weights, weight_seed=0)
    torch.cuda.synchronize()
    if a.prim == "bfs":
        from paper_1701_01170_b200.primitives.bfs import bfs_device

        fn = lambda: bfs_device(dg, 0, direction=a.direction)
    elif a.prim == "sssp":
        from paper_1701_01170_b200.primitives.sssp import sssp_device

        fn = lambda: sssp_device(dg, 0, delta=a.delta)
    elif a.prim == "pagerank":
        from paper_1701_01170_b200.primitives.pagerank import pagerank_device

        fn = lambda: (None, None, pagerank_device(dg, 0.85, 0.0, 20)[1])
    else:
        raise SystemExit(f"unknown primitive {a.prim}")
    if a.timing:
        dg.ctx.set_timing(True)
    for _ in range(a.warmup):
        fn()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.runs):
        st = fn()[2]
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("device_ms", st.device_ms, "E_r", getattr(st, "edges_reached", None), "init_ms",
          getattr(st, "init_ms", None), "loop_ms", getattr(st, "loop_ms", None))
    for lv in getattr(st, "device_levels", []):
        print("  ", lv)


if __name__ == "__main__":
    main()
