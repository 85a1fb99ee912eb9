nproc; free -g | head -2
python -m pytest tests/test_gpu_fullsize.py -q -x -k "alex32 or resnet50g" 2>&1 | tail -15 > gpurun_out/fs1.log
python -m pytest tests/test_gpu_training.py -q -k "device_stash" 2>&1 | tail -3 >> gpurun_out/fs1.log
timeout 900 python bench.py --pool-bytes 3905683456 --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r50_minpool.json 2> gpurun_out/bench_r50_minpool.err
timeout 900 python bench.py --pool-bytes 3905683456 --stash device --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r50_minpool_dev.json 2> gpurun_out/bench_r50_minpool_dev.err
python -m pytest tests/test_gpu_fullsize.py -q -k "not alex32 and not resnet50g" 2>&1 | tail -15 > gpurun_out/fs2.log
cat gpurun_out/fs1.log gpurun_out/fs2.log
