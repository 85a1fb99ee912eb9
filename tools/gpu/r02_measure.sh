# one call: the per-launch table at this build (ncu region + kernel census), merged on the box so
# bench.py finds a traffic file with the matching libsnexec digest, then the headline bench line
set -e
TAG=${TAG:-r02_resnet50g}
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/lt.csv python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt.json --ncu-region > gpurun_out/lt.log 2>&1
python tools/launch_table.py merge gpurun_out/lt.json gpurun_out/lt.csv --tag $TAG
cp profiles/${TAG}_launches.md profiles/${TAG}_step_traffic.json gpurun_out/
python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks']); print(json.dumps(d['roofline'])[:1500]); print(json.dumps(d['roofline_hbm_layers']))"
