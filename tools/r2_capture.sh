# final round-2 evidence: ncu of the ring at the bench's picks, sanitizers,
# GPU tests, smoke, full bench lines (driver command, default), reference arm
P=${1:-r2fin}
for gk in "20 20" "20 200"; do
  set -- $gk
  ncu --set full --import-source on --clock-control none -k regex:track_persist_kernel -s 1 -c 1 \
      -o gpurun_out/${P}_ring_g$1_k$2 python tools/ncu_ring.py $1 $2 > gpurun_out/${P}_ncu_g$1_k$2.log 2>&1
done
bash tools/run_sanitizers.sh > gpurun_out/${P}_sanitizers.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${P}_gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
bash tools/r2_final.sh ${P}
