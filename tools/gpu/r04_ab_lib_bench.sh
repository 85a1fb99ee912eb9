# A/B of two libsnexec builds (ablib/libsnexec_{old,new}.so) on the bench step time
L=paper_1801_04380_b200/_lib/libsnexec.so
for v in old new old new; do
  cp ablib/libsnexec_$v.so $L
  timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 --no-extras ${NET:+--net $NET} 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '${NET:-resnet50g}', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done
cp ablib/libsnexec_new.so $L
