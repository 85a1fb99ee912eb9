#!/bin/bash
out=gpurun_out/ncu_r04_stem
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:stem_rows_kernel|stem_wgrad_rows" -c 2 -o $out \
  python tools/profile_step.py --steps 1 > ${out}.log 2>&1
ncu -i ${out}.ncu-rep --page raw --csv > ${out}_raw.csv 2>/dev/null
python tools/ncu_summary.py report ${out}.ncu-rep > ${out}.md 2>/dev/null
ncu -i ${out}.ncu-rep --page source --csv --launch-count 1 > ${out}_src_fwd.csv 2>/dev/null
ncu -i ${out}.ncu-rep --page source --csv --launch-skip 1 --launch-count 1 > ${out}_src_wg.csv 2>/dev/null
ncu -i ${out}.ncu-rep --page details --csv > ${out}_details.csv 2>/dev/null
ls -la gpurun_out/ncu_r04_stem*
