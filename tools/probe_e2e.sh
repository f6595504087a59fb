# persistent-runner e2e vs H2D stream count (push mode)
for hs in 1 2 3; do
  FT_RUNNER_H2D_STREAMS=$hs timeout 300 python bench.py --quick --no-configs --steps 1000 --warmup 5 > gpurun_out/r2ak_h$hs.json 2>/dev/null
done
