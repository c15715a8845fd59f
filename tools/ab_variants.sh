# A/B of library build variants (build/ab/*.so, paper_2205_07307_b200.build.build_variant) on one box:
#   bash tools/ab_variants.sh OUT "c3 c2" lib1 lib2 ...   (interleaved, 2 rounds)
OUT=$1; CFGS=$2; shift 2
for round in 1 2; do for cfg in $CFGS; do for lib in "$@"; do
  if [ "$lib" = product ]; then python tools/time_kernels.py --config $cfg --reps 20 --tag product
  else ODF_LIB_OVERRIDE=$lib python tools/time_kernels.py --config $cfg --reps 20 --tag $(basename $lib .so); fi
done; done; done > gpurun_out/$OUT 2>&1
