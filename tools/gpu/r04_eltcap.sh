for c in 1184 888 592 444 296; do SN_ELT_CAP=$c python tools/kernel_grep.py 'bn_apply_v4|bn_dx_v4' > gpurun_out/eltcap_$c.txt 2>&1; tail -1 gpurun_out/eltcap_$c.txt; done
