"""Build kernel tuning variants into paper_1505_05571_b200/lib/variants/."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_05571_b200.build import build_variant  # noqa: E402

B = ("EXSUM_BUFFERS=1", "EXSUM_DECODE=2")
VARIANTS = {
    "v10_p1": B + ("EXSUM_VEC_PER_LANE=10", "EXSUM_PREFETCH_BATCHES=1"),
    "v12_p1": B + ("EXSUM_VEC_PER_LANE=12", "EXSUM_PREFETCH_BATCHES=1"),
    "v16_p1": B + ("EXSUM_VEC_PER_LANE=16", "EXSUM_PREFETCH_BATCHES=1"),
    "v12_p0": B + ("EXSUM_VEC_PER_LANE=12", "EXSUM_PREFETCH_BATCHES=0"),
    "v12_p1_g2": B + ("EXSUM_VEC_PER_LANE=12", "EXSUM_PREFETCH_BATCHES=1", "EXSUM_CHECK_GROUP=2"),
    "v12_p1_g4": B + ("EXSUM_VEC_PER_LANE=12", "EXSUM_PREFETCH_BATCHES=1", "EXSUM_CHECK_GROUP=4"),
    "v16_p1_g4": B + ("EXSUM_VEC_PER_LANE=16", "EXSUM_PREFETCH_BATCHES=1", "EXSUM_CHECK_GROUP=4"),
    "v10_p1_g2": B + ("EXSUM_VEC_PER_LANE=10", "EXSUM_PREFETCH_BATCHES=1", "EXSUM_CHECK_GROUP=2"),
}
names = sys.argv[1:] or list(VARIANTS)
verbose = "-v" in names
names = [n for n in names if n != "-v"] or list(VARIANTS)
for n in names:
    print(build_variant(n, VARIANTS[n], verbose=verbose))
