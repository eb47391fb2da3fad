"""Build a variant of the CUDA library for A/B timing (FFTC_LIB=... at run time).

  python scripts/build_ab.py NAME -DFFTC_SOMETHING=1 [...]

Objects go to build/ab_NAME/, the library to _ab/NAME/libfftcond_b200.so
(git-ignored, travels to the GPU box with the snapshot).
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2001_08289_b200 import build_ext as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
root = os.path.dirname(B.HERE)
B.BUILD = os.path.join(root, "build", f"ab_{name}")
os.makedirs(os.path.join(root, "_ab", name), exist_ok=True)
B.LIB = os.path.join(root, "_ab", name, "libfftcond_b200.so")
print(B.build(extra=extra))
