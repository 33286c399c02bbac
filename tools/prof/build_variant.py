"""Build a variant of libzkl_b200.so with extra nvcc defines (register /
occupancy experiments), next to the product build:

    python tools/prof/build_variant.py minb2 -DZKL_DENSE_MINB=2
    ZKL_LIB=build/variants/minb2/libzkl_b200.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, ".")
from paper_2508_21393_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
d = os.path.join("build", "variants", name)
os.makedirs(d, exist_ok=True)
print(B.build(extra_flags=flags, out=os.path.join(d, "libzkl_b200.so"),
              build_dir=os.path.join(d, "obj")))
