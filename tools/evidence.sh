# Round-1 evidence commands (run on a gpurun box from the repo root; outputs in gpurun_out/).
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 20 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:odf_main_kernel -c 3 -o gpurun_out/prof_c2 python tools/prof_kernels.py --config c2 --iters 1 > gpurun_out/ncu_full.log 2>&1
for cfg in c2 c3; do ODF_LIB_OVERRIDE=build/diag/libodf_t8.so python tools/timeline.py --config $cfg --mode fused; ODF_LIB_OVERRIDE=build/diag/libodf_t8.so python tools/timeline.py --config $cfg --mode apply; done > gpurun_out/timeline.jsonl 2>&1
for cfg in c2 c3 c4; do python tools/bench_formats.py --config $cfg; done > gpurun_out/formats.jsonl 2>&1
