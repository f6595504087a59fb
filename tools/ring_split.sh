for g in 1 0; do
  cp paper_2509_10757_b200/lib_gc$g.so paper_2509_10757_b200/libfasttrack_b200.so
  echo "== group claim $g"
  RING_R_MULT=140 RING_GROUPS=1,4,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
done
cp paper_2509_10757_b200/lib_gc1.so paper_2509_10757_b200/libfasttrack_b200.so
timeout 200 python tools/debug_pipe.py
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
