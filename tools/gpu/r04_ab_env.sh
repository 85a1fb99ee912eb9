# A/B of an environment variable: VAR with the values in VALS (step time, clocks), alternating
for v in ${VALS}; do
  env ${VAR}=$v python bench.py --steps 30 --warmup 5 --no-extras ${NET:+--net $NET} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('${VAR}=$v', d['ms_per_step'], d['value'], d['clocks'])"
done
