# round-3 evidence at this build: per-launch table (ncu region + kernel census,
# with the tensor-core SMEM operand metric), ncu --set full of the stage-1 halo
# kernels, then the headline bench line (reads the traffic file of this build)
set -e
TAG=${TAG:-r03_resnet50g}
M=$(python -c "import sys; sys.path.insert(0,'tools'); import launch_table as t; print(t.METRICS)")
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/lt.csv \
  python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt.json --ncu-region > gpurun_out/lt.log 2>&1
python tools/launch_table.py merge gpurun_out/lt.json gpurun_out/lt.csv --tag $TAG
cp profiles/${TAG}_launches.md profiles/${TAG}_step_traffic.json gpurun_out/
bash tools/ncu_capture.sh stage1 "tc_conv_halo_kernel|tc_conv_halo_wgrad64" 3 || true
python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value']); print(json.dumps(d['roofline'])[:1500]); print(json.dumps(d['roofline_hbm_layers']))"
