run warp_f602 ES_SPMM_KERNEL=warp -- --config reddit
for st in 4 8 16; do for r in 2 4 8 16 32; do
  run tma_f602_st${st}_r${r} ES_SPMM_STAGES=$st ES_SPMM_ROWS_PER_CTA=$r -- --config reddit
done; done
run warp_f128 ES_SPMM_KERNEL=warp -- --config reddit --F 128
for st in 8 16; do for r in 4 8 16 32; do
  run tma_f128_st${st}_r${r} ES_SPMM_STAGES=$st ES_SPMM_ROWS_PER_CTA=$r -- --config reddit --F 128
done; done
