#!/bin/bash
timeout 100 python tools/conv_bench.py --ops fwd --shapes 1 3 --halo 2 --pairs 0 1 > gpurun_out/r04_s2b_bench.txt 2>&1
SN_HALO_ES1=1 timeout 100 python tools/conv_bench.py --ops fwd --shapes 1 3 --halo 2 --pairs 0 1 >> gpurun_out/r04_s2b_bench.txt 2>&1
