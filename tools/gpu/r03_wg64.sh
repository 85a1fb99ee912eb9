# M=128 halo wgrad64 + split-K reduce + reverse BN dx: kernel tests, per-shape timing, step A/B
python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_fwd_dgrad_wgrad" 2>&1 | tail -3
for m in 1 0; do
  echo "SN_HALO_WG_M128=$m"; SN_HALO_WG_M128=$m python tools/conv_bench.py --pairs 1 --ops wgrad --shapes 0 2>&1 | tail -2
done
for env in "SN_XSKIP=0" "SN_HALO_WG_M128=0" "SN_XSKIP=256" "SN_XSKIP=0"; do
  env $env python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$env', d['ms_per_step'], d['value'], d['clocks'], d['losses'][-1])"
done
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
