for cfg in c3 c2 c4; do
  python tools/time_kernels.py --config $cfg --reps 10 --tag desc4
  ODF_LIB_OVERRIDE=build/ab/libodf_desc8.so python tools/time_kernels.py --config $cfg --reps 10 --tag desc8
done > gpurun_out/r2c_ab_desc.jsonl 2>&1
