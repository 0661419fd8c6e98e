P=paper_2511_05895_b200
cp $P/libdmf.so /tmp/libdmf_new.so
for v in nol1 new; do
  if [ $v = nol1 ]; then cp baseline_prev/libdmf_nol1.so $P/libdmf.so; else cp /tmp/libdmf_new.so $P/libdmf.so; fi
  for r in 1 2; do timeout 250 python tools/debug_smin.py 3 2>&1 | grep "^F" | sed "s/^/$v: /"; done
done
cp /tmp/libdmf_new.so $P/libdmf.so
