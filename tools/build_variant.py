"""Build a tuning variant of libtmotif.so: python tools/build_variant.py NAME -DKNOB=V ...
-> variants/NAME/libtmotif.so (git-ignored; travels to the GPU box with gpurun)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_02800_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
d = os.path.join(ROOT, "variants", name)
B.build(extra_flags=flags, lib=os.path.join(d, "libtmotif.so"), obj=os.path.join(d, "obj"))
print(os.path.join(d, "libtmotif.so"))
