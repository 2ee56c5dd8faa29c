"""Tuning A/B: build variants of the library with extra -D flags into
paper_2108_01731_b200/_lib/ab_<name>/ (selected at run time with
LCC_LIB_PATH).  Usage: python tools/ab_build.py name1='-DX=1 -DY=2' name2='...'"""
import os
import shlex
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2108_01731_b200 import build as B  # noqa: E402

for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = os.path.join(B.OUT_DIR, "ab_" + name)
    print(name, B.build(extra=shlex.split(flags), out_dir=out))
