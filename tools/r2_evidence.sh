# Round-2 evidence (run on a gpurun box from the repo root; outputs in gpurun_out/).
#   bash tools/r2_evidence.sh TAG [tests] [bench] [reference] [ncu] [launches] [extras]
TAG=${1:-r2}; shift
for step in "$@"; do case $step in
tests)
  python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" ;;
bench)
  python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" ;;
ncu)
  for cfg in c3 c2 c4; do
    ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 1 \
        -o gpurun_out/${TAG}_${cfg}_fused python tools/prof_kernels.py --config $cfg --iters 1 --only fused \
        > gpurun_out/${TAG}_ncu_${cfg}.log 2>&1; echo "ncu $cfg rc=$?"
  done
  ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 1 \
      -o gpurun_out/${TAG}_c3_binarize python tools/prof_kernels.py --config c3 --iters 1 --only binarize \
      > gpurun_out/${TAG}_ncu_c3_binarize.log 2>&1; echo "ncu c3 binarize rc=$?" ;;
reference)
  python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?" ;;
extras)
  python tools/bench_latency.py > gpurun_out/${TAG}_latency_c5.json 2> gpurun_out/${TAG}_latency.err; echo "latency rc=$?"
  python tools/bench_mixed.py > gpurun_out/${TAG}_mixed.json 2> gpurun_out/${TAG}_mixed.err; echo "mixed rc=$?"
  python tools/time_wide.py > gpurun_out/${TAG}_wide.json 2> gpurun_out/${TAG}_wide.err; echo "wide rc=$?" ;;
launches)
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 20 --warmup 3 \
      --secondary none --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launches rc=$?" ;;
esac; done
