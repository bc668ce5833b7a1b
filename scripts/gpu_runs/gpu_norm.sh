# one-step (chain-free) normalisation (EXSUM_NORM_PARALLEL)
mkdir -p gpurun_out/norm
P=gpurun_out/norm
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $P/tests.log 2>&1
timeout 1800 python scripts/ab_variants.py --cases c4,c3,c5 --rounds 4 default normseq > $P/time.log 2>&1
true
