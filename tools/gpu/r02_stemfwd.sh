python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -q -x -k "stem or resnet50g or alex32_matches or smoke or fusions" 2>&1 | tail -3
python tools/profile_step.py --steps 2 --order 2>/dev/null | grep -E " conv_stem| bn_stem" | head -4
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['clocks'])"; done
