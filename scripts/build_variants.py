"""Build kernel tuning variants into paper_1505_05571_b200/lib/variants/."""
import sys
from pathlib import Path

import importlib.util  # noqa: E402

# build.py by path: importing the package would load the library it builds
_spec = importlib.util.spec_from_file_location(
    "_exsum_b200_build", Path(__file__).resolve().parents[1] / "paper_1505_05571_b200" / "build.py")
_builder = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_builder)
build_variant = _builder.build_variant

VARIANTS = {
    "nofast": ("EXSUM_UNIFORM_FAST=0",),
    "backoff0": ("EXSUM_UNIFORM_BACKOFF=0",),
    "backoff15": ("EXSUM_UNIFORM_BACKOFF=15",),
    "timeline": ("EXSUM_TIMELINE=1",),
    "seg4": ("EXSUM_SEG_VEC=4",),
    "seg6": ("EXSUM_SEG_VEC=6",),
    "xorimad": ("EXSUM_XOR_LOP=0",),
    "cta132": ("EXSUM_MAX_CTAS=132",),
    "fullgrid": ("EXSUM_OVERLAP_SHORT=0",),
    "w8s65": ("EXSUM_RIPPLE=0", "EXSUM_SLOTS=65",),
    "w9v8": ("EXSUM_RIPPLE=0", "EXSUM_SLOTS=65", "EXSUM_WARPS=9"),
    "w9v7": ("EXSUM_RIPPLE=0", "EXSUM_SLOTS=65", "EXSUM_WARPS=9", "EXSUM_VEC_PER_LANE=7"),
    "w9v6": ("EXSUM_RIPPLE=0", "EXSUM_SLOTS=65", "EXSUM_WARPS=9", "EXSUM_VEC_PER_LANE=6"),
    "sumloop": ("EXSUM_SUM_SCAN=0",),
    "ldg1": ("EXSUM_LDG_KIND=1",),
    "ldg0": ("EXSUM_LDG_KIND=0",),
    "ldg3": ("EXSUM_LDG_KIND=3",),
    "ldg4": ("EXSUM_LDG_KIND=4",),
    "pf0": ("EXSUM_PREFETCH_BATCHES=0",),
    "pf2": ("EXSUM_PREFETCH_BATCHES=2",),
    "v6": ("EXSUM_VEC_PER_LANE=6",),
    "fixcg": ("EXSUM_FIX_L1=0",),
    "fixl1": ("EXSUM_FIX_L1=1",),
    "pfold": ("EXSUM_PF_ALIGNED=0",),
    "nomag": ("EXSUM_UNIFORM_SIGNED=0",),
    "debug": ("EXSUM_DEBUG_CHECKS=1",),
    "pfbranch": ("EXSUM_PF_PRED=0",),
    "segfix0": ("EXSUM_SEG_FIX_GROUP=0",),
    "segfix2": ("EXSUM_SEG_FIX_GROUP=2",),
    "segahead1": ("EXSUM_SEG_AHEAD=1",),
    "il0": ("EXSUM_INTERLEAVE=0",),
    "nodisp": ("EXSUM_UNIFORM_DISPATCH=0",),
    "onephase": ("EXSUM_TWO_PHASE=0",),
    "wimad": ("EXSUM_W_XOR_IMAD=1", "EXSUM_W_PLANES=1"),
    "oneplane": ("EXSUM_W_PLANES=1",),
    "ripple": ("EXSUM_RIPPLE=1",),
    "noripple": ("EXSUM_RIPPLE=0",),
    "rsplit": ("EXSUM_RIPPLE=1", "EXSUM_SEG_SPLIT=1"),
    "rseg8": ("EXSUM_RIPPLE=1", "EXSUM_SEG_VEC=8"),
    "rseg6": ("EXSUM_RIPPLE=1", "EXSUM_SEG_VEC=6"),
    "rv7": ("EXSUM_RIPPLE=1", "EXSUM_VEC_PER_LANE=7"),
    "rpf2": ("EXSUM_RIPPLE=1", "EXSUM_PREFETCH_BATCHES=2"),
    "rw10": ("EXSUM_RIPPLE=1", "EXSUM_WARPS=10"),
    "rsegfix0": ("EXSUM_RIPPLE=1", "EXSUM_SEG_FIX_GROUP=0"),
    "rv4": ("EXSUM_VEC_PER_LANE=4",),
    "rv5": ("EXSUM_VEC_PER_LANE=5",),
    "rseg5": ("EXSUM_SEG_VEC=5",),
    "sq3": ("EXSUM_SQNORM_VEC=3",),
    "sq8": ("EXSUM_SQNORM_VEC=8",),
    "sq5": ("EXSUM_SQNORM_VEC=5",),
    "dot4": ("EXSUM_DOT_VEC=4",),
    "dot3": ("EXSUM_DOT_VEC=3",),
    "rpf0": ("EXSUM_PREFETCH_BATCHES=0",),
    "rtp27": ("EXSUM_TWO_PHASE_MIN=(1ull<<26)",),
    "rpfnext": ("EXSUM_SEG_PF_NEXT=1",),
    "rsegahead": ("EXSUM_SEG_AHEAD=1",),
    "rnosplit": ("EXSUM_SEG_SPLIT=0",),
    "ripplev6": ("EXSUM_RIPPLE=1", "EXSUM_VEC_PER_LANE=6", "EXSUM_SEG_VEC=6"),
    "v7": ("EXSUM_VEC_PER_LANE=7",),
    "seg8": ("EXSUM_SEG_VEC=8",),
    "segtail2": ("EXSUM_SEG_TAIL=2",),
    "segtail8": ("EXSUM_SEG_TAIL=8",),
}
names = sys.argv[1:] or list(VARIANTS)
verbose = "-v" in names
names = [n for n in names if n != "-v"] or list(VARIANTS)
for n in names:
    print(build_variant(n, VARIANTS[n], verbose=verbose))
