python tools/precision_probe.py > gpurun_out/prec2.txt 2>&1
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -q -x -k "3xtf32 or fp32 or pool_bn or fusions" 2>&1 | tail -4 >> gpurun_out/prec2.txt
python -m pytest tests/test_gpu_fullsize.py -q -k "resnet2534g or densenet or resnet50g" 2>&1 | tail -5 >> gpurun_out/prec2.txt
timeout 600 python bench.py --steps 5 --warmup 3 --precision fp32 --no-extras > gpurun_out/bench_fp32.json 2>gpurun_out/bench_fp32.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err
cat gpurun_out/prec2.txt
