python -m pytest tests/test_gpu_training.py -q -x -k "pipelined or host" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
python -c "import json; d=json.loads(open('gpurun_out/b_e2e.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks']); print(json.dumps(d['e2e']))"
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
