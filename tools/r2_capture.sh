# ncu --set full of the bench's value kernel (ring) at the step-group counts
# the bench picks (10 at K=20, 14 at K=200), the launch list of the driver's
# bench command, then compute-sanitizer on every kernel
P=${1:-r2x}
for gk in "10 20" "14 200" "1 20"; do
  set -- $gk
  ncu --set full --import-source on --clock-control none -k regex:track_persist_kernel -s 1 -c 1 \
      -o gpurun_out/${P}_ring_g$1_k$2 python tools/ncu_ring.py $1 $2 > gpurun_out/${P}_ncu_g$1_k$2.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --steps 20 --warmup 5 --quick > gpurun_out/${P}_launches_bench.log 2>&1
bash tools/run_sanitizers.sh > gpurun_out/${P}_sanitizers.txt 2>&1
