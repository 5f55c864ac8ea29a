"""Grid-barrier cost on this GPU: cooperative-groups grid sync vs the flag
barrier, for the persistent BFS kernel's grid shapes."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_01170_b200 import _native  # noqa: E402

ctx = _native.Context(0)
for blocks, threads in ((444, 256), (296, 256), (148, 768), (148, 256), (148, 512)):
    for variant in (0, 1, 2, 3):
        us = ctypes.c_float()
        _native.call("gfx_debug_gridsync", ctx.handle, variant, blocks, threads, 2000,
                     ctypes.byref(us))
        print(f"blocks {blocks:4d} x {threads:4d}  {('cg', 'flag', 'cg+ctr-all', 'cg+ctr-t0')[variant]}  "
              f"{us.value:.3f} us/sync")

# same-address atomics (one per warp per iteration): the level counters'
# serialisation cost
for variant, name in ((0, "same address, returned"), (1, "same address, RED"),
                      (2, "own line per warp")):
    for blocks in (148, 444):
        ns = ctypes.c_double()
        _native.call("gfx_debug_atomics", ctx.handle, variant, blocks, 50, ctypes.byref(ns))
        print(f"atomics {name:24s} blocks {blocks:4d}: {ns.value:.3f} ns per atomic "
              f"({ns.value * blocks * 8 / 1000:.2f} us per round of {blocks * 8} warps)")
