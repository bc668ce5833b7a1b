"""Build kernel tuning variants into paper_1505_05571_b200/lib/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200.build import build_variant  # noqa: E402

VARIANTS = {
    "v8": ("EXSUM_VEC_PER_LANE=8",),
    "v9": ("EXSUM_VEC_PER_LANE=9",),
    "v10": ("EXSUM_VEC_PER_LANE=10",),
    "v12": ("EXSUM_VEC_PER_LANE=12",),
    "v8_p2": ("EXSUM_VEC_PER_LANE=8", "EXSUM_PREFETCH_BATCHES=2"),
    "v10_p2": ("EXSUM_VEC_PER_LANE=10", "EXSUM_PREFETCH_BATCHES=2"),
}
names = sys.argv[1:] or list(VARIANTS)
verbose = "-v" in names
names = [n for n in names if n != "-v"] or list(VARIANTS)
for n in names:
    print(build_variant(n, VARIANTS[n], verbose=verbose))
