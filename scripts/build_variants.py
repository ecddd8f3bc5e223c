"""Build tuning variants of libadop.so (scratch, git-ignored .so files): python scripts/build_variants.py NAME=DEFS..."""
import sys

sys.path.insert(0, ".")
from paper_2110_06635_b200 import build as B  # noqa: E402

for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    out = f"paper_2110_06635_b200/libadop_{name}.so"
    B.build(out=out, defines=[d for d in defs.split(",") if d])
    print("built", out)
