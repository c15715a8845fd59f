timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in c2 c3 c4; do python tools/time_kernels.py --config $cfg --tag ndl4; done
