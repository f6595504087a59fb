# ncu --set full of the bench's value kernel (ring) per step-group count, the
# launch list of the default bench command, then compute-sanitizer on every
# kernel (tools/run_sanitizers.sh)
P=${1:-r2n}
for gk in "8 20" "4 20" "1 20" "8 200"; do
  set -- $gk
  ncu --set full --import-source on --clock-control none -k regex:track_persist_kernel -s 1 -c 1 \
      -o gpurun_out/${P}_ring_g$1_k$2 python tools/ncu_ring.py $1 $2 > gpurun_out/${P}_ncu_g$1_k$2.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --steps 20 --warmup 5 --quick > gpurun_out/${P}_launches_bench.log 2>&1
bash tools/run_sanitizers.sh > gpurun_out/${P}_sanitizers.txt 2>&1
