"""Build A/B variants of libmpxa (compile-time -D switches) into paper_2309_07337_b200/variants/.
Usage: python tools/build_variants.py NAME=DEFINE[,DEFINE...] ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_07337_b200 import _build
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    out = os.path.join(_build.HERE, "variants", f"libmpxa_{name}.so")
    _build.build(force=True, defines=tuple(d for d in defs.split(",") if d), out=out)
    print(out)
