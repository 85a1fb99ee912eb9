python -m pytest tests/test_gpu_training.py tests/test_gpu_kernels.py -q -x -k "stem or fusions or bit_identical or resnet50g or fp32_mode" 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fused', d['value'], d['ms_per_step'], d['clocks'])"
SN_FUSE_STEM_BN=0 python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('unfused', d['value'], d['ms_per_step'], d['clocks'])"
done
python tools/profile_step.py --steps 2 --order 2>/dev/null | grep -E "bn_stem|conv_stem|conv_s2b1" | head -8
SN_FUSE_STEM_BN=0 python tools/profile_step.py --steps 2 --order 2>/dev/null | grep -E "bn_stem|conv_stem|conv_s2b1" | head -8
