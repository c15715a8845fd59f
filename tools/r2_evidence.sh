# Round-2 evidence (run on a gpurun box from the repo root; outputs in gpurun_out/).
#   bash tools/r2_evidence.sh TAG [tests] [bench] [ncu] [launches]
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
  done ;;
launches)
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 20 --warmup 3 \
      --secondary none --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launches rc=$?" ;;
esac; done
