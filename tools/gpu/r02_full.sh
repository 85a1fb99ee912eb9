# full GPU suite, smoke, headline bench, depth / floor configs (bench lines under gpurun_out/)
python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/full_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
timeout 900 python bench.py --net resnet2534g --steps 5 --warmup 3 --no-extras > gpurun_out/bench_r2534.json 2> gpurun_out/bench_r2534.err
timeout 900 python bench.py --net resnet152g --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r152.json 2> gpurun_out/bench_r152.err
timeout 900 python bench.py --pool-bytes 3288334336 --steps 10 --warmup 3 --no-extras > gpurun_out/bench_r50_floor.json 2> gpurun_out/bench_r50_floor.err
cat gpurun_out/full_tests.log
tail -2 gpurun_out/*.err
