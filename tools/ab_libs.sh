# A/B of library builds on the resident ring: bash tools/ab_libs.sh TAG lib1 lib2 ...
# (each build/libX.so replaces the in-tree library in turn, twice, interleaved;
# ring_groups.py checks parity against the oracle after every configuration)
TAG=$1; shift
cp paper_2509_10757_b200/libfasttrack_b200.so build/lib_intree.so
for rep in 1 2; do
  for L in "$@"; do
    cp build/lib$L.so paper_2509_10757_b200/libfasttrack_b200.so
    echo "== $L rep $rep" >> gpurun_out/${TAG}_ab.txt
    RING_R_MULT=140 RING_GROUPS=${RING_GROUPS:-10,14} timeout 300 python tools/ring_groups.py >> gpurun_out/${TAG}_ab.txt 2>&1
  done
done
cp build/lib_intree.so paper_2509_10757_b200/libfasttrack_b200.so
cat gpurun_out/${TAG}_ab.txt
