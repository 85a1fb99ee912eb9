# final evidence of the round at this build: per-launch table + digest-stamped
# traffic (the headline bench reads it), the other BASELINE configs, then the
# default headline bench after a cool-down
TAG=r04_resnet50g
M=$(python -c "import sys; sys.path.insert(0,'tools'); import launch_table as t; print(t.METRICS)")
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/lt.csv \
  python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt.json --ncu-region > gpurun_out/lt.log 2>&1
python tools/launch_table.py merge gpurun_out/lt.json gpurun_out/lt.csv --tag $TAG
cp profiles/${TAG}_launches.md profiles/${TAG}_step_traffic.json gpurun_out/
for net in alex32 resnet152g densenet121s inception4s resnet2534g; do
  timeout 1200 python bench.py --net $net --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r04_$net.json 2> gpurun_out/bench_r04_$net.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r04_$net.json').read().strip().splitlines()[-1]); print('$net', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'])"
done
sleep 30
python bench.py > gpurun_out/bench_r04_resnet50g.json 2> gpurun_out/bench_r04_resnet50g.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r04_resnet50g.json').read().strip().splitlines()[-1]); print('resnet50g', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic_source'])"
