#!/bin/bash
for v in 0 3 4 5; do echo "S2V=$v"; SN_HALO_S2V=$v timeout 100 python tools/conv_bench.py --ops fwd --shapes 1 --halo 2 --pairs 1 2>&1; done > gpurun_out/r04_s2c_bench.txt
