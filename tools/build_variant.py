"""Build a tuning variant of libbfapply.so with extra -D defines:  python tools/build_variant.py NAME DEF1 [DEF2 ...]
-> tools/variants/lib_NAME.so (git-ignored; travels to the GPU box).  Experiments only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
name, defs = sys.argv[1], sys.argv[2:]
from paper_1803_04128_b200 import build as B  # noqa: E402

B.NVCC_FLAGS += [f"-D{d}" for d in defs]
print(B.build(out=os.path.join(ROOT, "tools", "variants", f"lib_{name}.so")))
