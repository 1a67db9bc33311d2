"""Build an A/B variant of the library with extra nvcc defines (measurement only).

  python tools/build_variant.py libchimera_x.so -DCHM_QA_POLY=0 [-DNAME=V ...]

writes paper_2603_22206_b200/<name> (objects under _build_<stem>/); select it
at run time with CHM_LIB=paper_2603_22206_b200/<name>."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_22206_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.NVCC_FLAGS = B.NVCC_FLAGS + defs
B.BUILD_DIR = os.path.join(B.HERE, "_build_" + name.rsplit(".", 1)[0])
B.LIB_PATH = os.path.join(B.HERE, name)
print(B.build(force=True))
