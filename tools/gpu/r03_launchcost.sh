# real cost of small launches in the captured step: idempotent kernels issued twice
for m in 0 512 1024 1536 0 512 1024 1536; do
  SN_XSKIP=$m python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/lc.json 2> gpurun_out/lc.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/lc.json').read().strip().splitlines()[-1]); print('mask $m', d['ms_per_step'], d['value'], d['clocks'], d['gpu_launches'])"
done
