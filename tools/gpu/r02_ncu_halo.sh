ncu --set full --clock-control none --import-source on -k "regex:tc_conv_halo_kernel<64" -c 1 -o gpurun_out/halo64 python tools/profile_step.py --steps 1 > gpurun_out/halo64.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tc_conv_halo_wgrad64" -c 1 -o gpurun_out/hwg64 python tools/profile_step.py --steps 1 > gpurun_out/hwg64.log 2>&1
ls -la gpurun_out/*.ncu-rep
