#!/usr/bin/env bash
# ncu --set full capture of the kernels matching $2 in one eager training step,
# exported on the box to CSV (raw metrics + per-kernel summary) so that only
# small files travel back.   usage: tools/ncu_capture.sh <tag> <regex> [count] [extra profile_step args]
set -u
tag=$1; rx=$2; cnt=${3:-8}; shift 3 || shift $#
out=gpurun_out/ncu_${tag}
ncu --set full --clock-control none --import-source on -k "regex:${rx}" -c "$cnt" -o "$out" \
    python tools/profile_step.py --steps 1 "$@" > "${out}.log" 2>&1
echo "ncu rc=$?"
ncu -i "${out}.ncu-rep" --page raw --csv > "${out}_raw.csv" 2>/dev/null
python tools/ncu_summary.py report "${out}.ncu-rep" > "${out}.md" 2>/dev/null
sz=$(stat -c %s "${out}.ncu-rep" 2>/dev/null || echo 0)
if [ "$sz" -gt 20000000 ]; then rm -f "${out}.ncu-rep"; echo "dropped ${out}.ncu-rep ($sz bytes)"; fi
