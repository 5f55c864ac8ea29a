"""Build a variant of libgfx.so with extra nvcc defines, for A/B runs
(GFX_LIB_PATH=paper_1701_01170_b200/libgfx_<name>.so).

    python tools/build_variant.py timeline -DGFX_BFS_TIMELINE
    python tools/build_variant.py head            # the tree as it is now
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_01170_b200 import _build  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    _build.NVCC_FLAGS = _build.NVCC_FLAGS + defs
    _build.BUILD = _build.PKG / f"_objs_{name}"
    _build.OUT = _build.PKG / f"libgfx_{name}.so"
    print(_build.build(verbose=False))


if __name__ == "__main__":
    main()
