ncu --set full --clock-control none --import-source on -k "regex:tc_conv_tma_kernel" -s 19 -c 1 -o gpurun_out/wg_s3 python tools/profile_step.py --steps 1 > gpurun_out/wg_s3.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tc_conv_tma_kernel" -s 20 -c 1 -o gpurun_out/dg_s3 python tools/profile_step.py --steps 1 > gpurun_out/dg_s3.log 2>&1
ls -la gpurun_out/*_s3.ncu-rep
