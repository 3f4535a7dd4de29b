"""Build a variant of the library with extra nvcc flags for A/B runs:
    python tools/build_variant.py NAME -DFLAG ...   ->  paper_1803_00430_b200/libechoforge_b200_NAME.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_00430_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
print(b.compile_library(b.LIB.replace(".so", f"_{name}.so"), flags))
