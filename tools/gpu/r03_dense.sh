python -m pytest tests/test_gpu_training.py -q -x -k "dense_join or branchy" 2>&1 | tail -3
for env in "SN_FUSE_DENSE=1" "SN_FUSE_DENSE=0" "SN_FUSE_DENSE=1"; do
  env $env python bench.py --net densenet121s --steps 10 --warmup 3 --no-extras > gpurun_out/bd.json 2> gpurun_out/bd.err
  python -c "import json; d=json.loads(open('gpurun_out/bd.json').read().strip().splitlines()[-1]); print('$env', d['value'], d['ms_per_step'], d['clocks'], d['gpu_launches'])"
done
