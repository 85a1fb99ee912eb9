# A/B of two libsnexec builds (ablib/libsnexec_{old,new}.so): kernel events of REGEX and step time
L=paper_1801_04380_b200/_lib/libsnexec.so
for v in old new old new; do
  cp ablib/libsnexec_$v.so $L
  echo "== $v"; python tools/kernel_grep.py "${REGEX}" ${NET:+--net $NET} | tail -${TAILN:-1}
done
cp ablib/libsnexec_new.so $L
