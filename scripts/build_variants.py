"""Build kernel tuning variants into paper_1505_05571_b200/lib/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200.build import build_variant  # noqa: E402

R = ("EXSUM_ROLL=1",)
VARIANTS = {
    "roll_v6": R + ("EXSUM_VEC_PER_LANE=6",),
    "roll_v5": R + ("EXSUM_VEC_PER_LANE=5",),
    "roll_v4": R + ("EXSUM_VEC_PER_LANE=4",),
    "roll_v3": R + ("EXSUM_VEC_PER_LANE=3",),
    "roll_v4_p2": R + ("EXSUM_VEC_PER_LANE=4", "EXSUM_PREFETCH_BATCHES=2"),
    "roll_v4_p3": R + ("EXSUM_VEC_PER_LANE=4", "EXSUM_PREFETCH_BATCHES=3"),
    "roll_v6_p2": R + ("EXSUM_VEC_PER_LANE=6", "EXSUM_PREFETCH_BATCHES=2"),
    "roll_v2_p4": R + ("EXSUM_VEC_PER_LANE=2", "EXSUM_PREFETCH_BATCHES=4"),
}
names = sys.argv[1:] or list(VARIANTS)
verbose = "-v" in names
names = [n for n in names if n != "-v"] or list(VARIANTS)
for n in names:
    print(build_variant(n, VARIANTS[n], verbose=verbose))
