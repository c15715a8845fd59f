# TMA streaming probe sweep (build first: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_probe tools/stream_probe.cu -lcuda).
for cfg in "2 2 128" "3 2 128" "2 1 128" "4 1 128" "6 1 128" "8 1 128" "12 1 128" "4 2 128" "6 2 128" "3 4 128" "4 1 256" "6 1 256" "8 1 64" "12 1 64"; do
  build/stream_probe 100000 1000 $cfg
done
for cfg in "2 2 128" "6 1 128" "12 1 128" "6 2 128"; do build/stream_probe 1000000 1000 $cfg; done
