"""Build TMA-pipeline tuning variants of libmpxa into paper_2309_07337_b200/variants/."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_07337_b200 import _build
VARIANTS = [(6, 16384, 4), (4, 32768, 2), (8, 8192, 6), (3, 32768, 1), (12, 8192, 9), (6, 16384, 3), (6, 16384, 5)]
for s, c, a in VARIANTS:
    out = os.path.join(_build.HERE, "variants", f"libmpxa_S{s}_C{c}_A{a}.so")
    _build.build(force=True, defines=(f"MPXA_STAGES={s}", f"MPXA_CHUNK={c}", f"MPXA_AHEAD={a}"), out=out)
    print(out)
