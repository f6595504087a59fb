# Ring value vs the stereo / map split: FT_GEOM_GM forces the map blocks per
# frame (the rest of a group's blocks run stereo); bash tools/ring_split_sweep.sh TAG
TAG=$1
for G in 10 14; do
  for GM in ${GMS:-2 3 4 5 6 7}; do
    echo "== G=$G Gm=$GM" >> gpurun_out/${TAG}_split.txt
    FT_GEOM_GM=$GM RING_R_MULT=140 RING_GROUPS=$G timeout 300 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY\|Error" >> gpurun_out/${TAG}_split.txt
  done
  echo "== G=$G model split" >> gpurun_out/${TAG}_split.txt
  RING_R_MULT=140 RING_GROUPS=$G timeout 300 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY" >> gpurun_out/${TAG}_split.txt
done
cat gpurun_out/${TAG}_split.txt
