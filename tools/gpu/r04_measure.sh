# round-4 evidence at this build: per-launch table (ncu region + kernel census),
# ncu --set full of the kernels changed this round, the headline bench line
# (reads the traffic file of this build) and the other BASELINE configs
TAG=${TAG:-r04_resnet50g}
M=$(python -c "import sys; sys.path.insert(0,'tools'); import launch_table as t; print(t.METRICS)")
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/lt.csv \
  python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt.json --ncu-region > gpurun_out/lt.log 2>&1
python tools/launch_table.py merge gpurun_out/lt.json gpurun_out/lt.csv --tag $TAG
cp profiles/${TAG}_launches.md profiles/${TAG}_step_traffic.json gpurun_out/
bash tools/ncu_capture.sh r04_step "tc_conv_halo_kernel|pool_fwd_k3s2|splitk_reduce|stem_rows" 12 || true
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r04_resnet50g.json 2> gpurun_out/bench_r04_resnet50g.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r04_resnet50g.json').read().strip().splitlines()[-1]); print('resnet50g', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value']); print(json.dumps(d['roofline'])[:800])"
for net in alex32 resnet152g densenet121s inception4s resnet2534g; do
  timeout 1200 python bench.py --net $net --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r04_$net.json 2> gpurun_out/bench_r04_$net.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r04_$net.json').read().strip().splitlines()[-1]); print('$net', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'])"
done
