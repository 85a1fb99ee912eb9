python -m pytest tests -m gpu -q 2>&1 | tail -12 > gpurun_out/suite.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/suite.log 2>&1
cat gpurun_out/suite.log
