"""Build experiment variants of libdot_b200.so into tools/variants/ (never
the product library): python tools/build_variants.py NAME=DEF1,DEF2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_15333_b200.build import build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
os.makedirs(OUT, exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    path = build(force=True, out=os.path.join(OUT, f"lib_{name}.so"), defines=[d for d in defs.split(",") if d])
    print(path)
