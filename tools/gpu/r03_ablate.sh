# A/B ablation of launch classes in the captured step (SN_XSKIP bitmask, see kernels.hpp)
for m in 0 1 2 3 4 8 16 32 64 96 128 0; do
  SN_XSKIP=$m python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/ab_$m.json 2> gpurun_out/ab_$m.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$m.json').read().strip().splitlines()[-1]); print('mask $m', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done
