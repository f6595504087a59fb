timeout 300 python -m pytest tests/test_gpu_pipeline.py -x -q -k "persistent" > gpurun_out/r2m_tests.log 2>&1; tail -1 gpurun_out/r2m_tests.log
for rep in 1 2; do
timeout 300 python bench.py --quick --no-configs --steps 1000 --warmup 5 > gpurun_out/r2m_push2_$rep.json 2>/dev/null
done
