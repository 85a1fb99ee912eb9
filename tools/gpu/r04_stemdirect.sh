SN_STEM_DIRECT=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -q -x -k "stem or resnet50g or fusions" 2>&1 | tail -2
for v in 0 1 0 1; do SN_STEM_DIRECT=$v python tools/kernel_grep.py "stem_rows" | tail -1; done
VAR=SN_STEM_DIRECT VALS="0 1 0 1" bash tools/gpu/r04_ab_env.sh
