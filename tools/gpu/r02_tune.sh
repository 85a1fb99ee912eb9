python -m pytest tests/test_gpu_training.py -q -x -k "autotune" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('default', d['value'], d['ms_per_step'], d['clocks'])"
python bench.py --steps 20 --warmup 5 --no-extras --autotune > gpurun_out/bench_tune.json; python -c "import json,sys; d=json.loads(open('gpurun_out/bench_tune.json').read().strip().splitlines()[-1]); print('autotune', d['value'], d['ms_per_step'], d['clocks'], d['autotune_catalog'])"
python bench.py --steps 20 --warmup 5 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('default', d['value'], d['ms_per_step'], d['clocks'])"
