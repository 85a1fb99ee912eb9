# round-3 bench lines: headline (full extras) and the other BASELINE configs
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r03_resnet50g.json 2> gpurun_out/bench_r03_resnet50g.err
python -c "import json; d=json.loads(open('gpurun_out/bench_r03_resnet50g.json').read().strip().splitlines()[-1]); print('resnet50g', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], json.dumps(d['unconstrained']))"
for net in alex32 resnet152g densenet121s inception4s resnet2534g; do
  timeout 1200 python bench.py --net $net --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r03_$net.json 2> gpurun_out/bench_r03_$net.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r03_$net.json').read().strip().splitlines()[-1]); print('$net', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'])"
done
