set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/t5.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/t5.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/b5.json 2> gpurun_out/b5.err
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/lt_r50.csv python tools/launch_table.py collect --net resnet50g --out gpurun_out/lt_r50.json --ncu-region > gpurun_out/lt_r50.log 2>&1
tail -3 gpurun_out/lt_r50.log
cat gpurun_out/t5.log
