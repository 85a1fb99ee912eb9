python -m pytest tests/test_gpu_fanjoin.py -q 2>&1 | tail -2
for net in alex32 densenet121s inception4s; do
  timeout 900 python bench.py --net $net --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r02_$net.json 2> gpurun_out/bench_r02_$net.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r02_$net.json').read().strip().splitlines()[-1]); print('$net', d['value'], d['ms_per_step'], d['clocks'])"
done
bash tools/ncu_capture.sh r02_bnbwd "colred_stage1_v4|bn_dx_v4" 6 > /dev/null 2>&1
bash tools/ncu_capture.sh r02_stem "stem_rows_kernel|stem_wgrad_rows_kernel|pool_fwd_k3s2" 3 > /dev/null 2>&1
bash tools/ncu_capture.sh r02_conv "tc_conv_halo_kernel|tc_conv_tma_kernel|tc_conv_halo_wgrad" 10 > /dev/null 2>&1
ls -la gpurun_out/ncu_r02_*
