# ncu shared-store conflict counters of the sum kernel (config 3) per library variant: VARIANTS="default rmw1" bash scripts/ncu_variants.sh
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset EXSUM_LIB; else export EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so; fi
  echo "== $v"
  ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,gpu__time_duration.sum --clock-control none -k regex:exsum_sum_kernel -s 1 -c 1 python scripts/prof_sum.py 3 1e8 2 2>&1 | grep -E "l1tex|gpu__time"
done
unset EXSUM_LIB
