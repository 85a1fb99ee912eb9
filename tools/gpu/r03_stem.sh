python -m pytest tests/test_gpu_kernels.py -q -x -k "stem" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:stem_rows_kernel" -c 2 python tools/profile_step.py --steps 1 2>&1 | grep -E "stem_rows|duration|tensor" | head -8
python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/bs.json 2> gpurun_out/bs.err
python -c "import json; d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks'])"
python -m pytest tests/test_gpu_training.py -q -x 2>&1 | tail -2
