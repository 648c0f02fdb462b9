"""Build A/B experiment variants of the library with extra -D flags.

    python scripts/variants.py NAME=DEF1,DEF2 [NAME2=...]
then run with MFREG_LIB_VARIANT=NAME (the package loads build/NAME/libmfreg_cuda_NAME.so).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_10541_b200._build import build  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    print(build(variant=name, defines=tuple(d for d in defs.split(",") if d)))
