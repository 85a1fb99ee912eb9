#!/bin/bash
# stride-2 phase-mode halo forward: parity + A/B timing
set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k "conv_fwd_dgrad_wgrad" > gpurun_out/r04_s2_test.log 2>&1
echo rc=$? >> gpurun_out/r04_s2_test.log
timeout 200 python tools/conv_bench.py --ops fwd --shapes 1 3 5 --halo 0 2 --pairs 0 1 > gpurun_out/r04_s2_bench.txt 2>&1
