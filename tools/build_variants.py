"""Build testing-library variants with extra -D flags for A/B timing on one box (diagnostics).
    python tools/build_variants.py NAME=-DFLAG=1[,-DFLAG2=..] ...   -> paper_2402_05099_b200/libhydra_var_NAME.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_05099_b200 import build as hb

for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    lib = os.path.join(hb.PKG, f"libhydra_var_{name}.so")
    hb._build_one(lib, hb.BUILD + f"_var_{name}", ["-DHYDRA_TESTING"] + flags.split(","), True, False, [])
    print(lib)
