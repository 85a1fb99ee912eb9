NCCL_DEBUG=WARN python tools/dp_check.py > gpurun_out/t8a.log 2>&1
NCCL_DEBUG=WARN python tools/dp_check.py eager > gpurun_out/t8b.log 2>&1
tail -30 gpurun_out/t8a.log; tail -30 gpurun_out/t8b.log
