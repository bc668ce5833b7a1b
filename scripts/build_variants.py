"""Build kernel tuning variants into paper_1505_05571_b200/lib/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200.build import build_variant  # noqa: E402

VARIANTS = {
    "d0": ("EXSUM_DECODE=0", "EXSUM_PIPE=0", "EXSUM_VEC_PER_LANE=8", "EXSUM_PREFETCH_BATCHES=1"),
    "d1": ("EXSUM_DECODE=1", "EXSUM_PIPE=0", "EXSUM_VEC_PER_LANE=8", "EXSUM_PREFETCH_BATCHES=1"),
    "d1_p1": ("EXSUM_DECODE=1", "EXSUM_PIPE=1", "EXSUM_VEC_PER_LANE=8", "EXSUM_PREFETCH_BATCHES=1"),
    "d1_p2": ("EXSUM_DECODE=1", "EXSUM_PIPE=2", "EXSUM_VEC_PER_LANE=8", "EXSUM_PREFETCH_BATCHES=1"),
}
names = sys.argv[1:] or list(VARIANTS)
verbose = "-v" in names
names = [n for n in names if n != "-v"] or list(VARIANTS)
for n in names:
    print(build_variant(n, VARIANTS[n], verbose=verbose))
