# Round-2 baseline captures (run on a gpurun box from the repo root).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_base_bench_c3.json 2> gpurun_out/r2_base_bench_c3.err
python tools/time_kernels.py --config c4 --reps 5 > gpurun_out/r2_base_time_c4.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 1 -o gpurun_out/r2_base_c3_fused python tools/prof_kernels.py --config c3 --iters 1 --only fused > gpurun_out/r2_base_ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 1 -o gpurun_out/r2_base_c4_fused python tools/prof_kernels.py --config c4 --iters 1 --only fused > gpurun_out/r2_base_ncu_c4.log 2>&1
ls -la gpurun_out
