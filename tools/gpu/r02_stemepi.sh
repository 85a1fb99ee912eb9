set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "stem" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -q -x 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', d['value'], d['ms_per_step'], d['clocks'])"
done
bash tools/gpu/r02_kbreak.sh; head -16 gpurun_out/kbreak.txt
