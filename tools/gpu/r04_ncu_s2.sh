#!/bin/bash
# ncu --set full of conv_s2b1 forward: im2col CTA-pair kernel vs stride-2 phase-mode halo kernel
out=gpurun_out/ncu_r04_s2
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tc_conv" -c 6 -o $out \
  python tools/conv_bench.py --ops fwd --shapes 1 --halo 0 2 --pairs 1 --iters 1 > ${out}.log 2>&1
ncu -i ${out}.ncu-rep --page raw --csv > ${out}_raw.csv 2>/dev/null
python tools/ncu_summary.py report ${out}.ncu-rep > ${out}.md 2>/dev/null
ncu -i ${out}.ncu-rep --page source --csv --launch-skip 5 --launch-count 1 > ${out}_src_halo.csv 2>/dev/null
ncu -i ${out}.ncu-rep --page source --csv --launch-skip 2 --launch-count 1 > ${out}_src_im2col.csv 2>/dev/null
ls -la gpurun_out/ncu_r04_s2*
