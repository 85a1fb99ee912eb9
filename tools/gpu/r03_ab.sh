# A/B of the SN_XSKIP options given in $MASKS (step time, clocks)
for m in ${MASKS:-0 2048 0 2048}; do
  SN_XSKIP=$m python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('mask $m', d['ms_per_step'], d['value'], d['clocks'])"
done
