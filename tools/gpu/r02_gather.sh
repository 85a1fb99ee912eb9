# stem pool-backward gather: correctness (bit identity) then A/B step time
set -x
python -m pytest tests/test_gpu_training.py -q -x -k "stem or bit_identical or fusions or resnet50g" 2>&1 | tail -5
python -m pytest tests/test_gpu_kernels.py -q -x -k "bn or pool or stem" 2>&1 | tail -3
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gather', d['value'], d['ms_per_step'], d['clocks'])"
SN_FUSE_POOL_GATHER=0 python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nogather', d['value'], d['ms_per_step'], d['clocks'])"
done
python tools/profile_step.py --steps 2 --order 2>/dev/null | grep -E "bn_stem|pool_stem|conv_stem" | head -6
SN_FUSE_POOL_GATHER=0 python tools/profile_step.py --steps 2 --order 2>/dev/null | grep -E "bn_stem|pool_stem|conv_stem" | head -6
