"""Builds tuning variants of libgt.so (A/B experiments): tools/variants/<name>/libgt.so."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16715_b200 import _build  # noqa: E402

VARIANTS = {}
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    VARIANTS[name] = [d for d in defs.split(",") if d]

for name, defs in VARIANTS.items():
    d = os.path.join(ROOT, "tools", "variants", name)
    os.makedirs(d, exist_ok=True)
    print(name, _build.build(defines=defs, lib=os.path.join(d, "libgt.so"), objdir=os.path.join(d, "obj")))
