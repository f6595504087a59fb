for l in 8 16 32; do
  cp paper_2509_10757_b200/lib_lpp$l.so paper_2509_10757_b200/libfasttrack_b200.so
  echo "== lanes per point $l"
  RING_R_MULT=140 RING_GROUPS=4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
done
cp paper_2509_10757_b200/lib_lpp16.so paper_2509_10757_b200/libfasttrack_b200.so
