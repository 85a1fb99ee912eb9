# ncu --set full of the stage-1 halo weight gradient (both MMA shapes) and the stem forward
set -u
for m in 1 0; do
  SN_HALO_WG_M128=$m ncu --set full --clock-control none --import-source on -k "regex:wgrad64|splitk" -c 4 -o gpurun_out/ncu_wg64_m$m \
    python tools/conv_bench.py --pairs 1 --ops wgrad --shapes 0 --iters 1 > gpurun_out/ncu_wg64_m$m.log 2>&1
  echo "m=$m rc=$?"
done
bash tools/ncu_capture.sh stemfwd "stem_rows_kernel" 1
ls -la gpurun_out/*.ncu-rep
