# GPU check used during round 2: the whole -m gpu suite, then quick bench lines
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$1_gputest.log 2>&1
tail -3 gpurun_out/$1_gputest.log
timeout 300 python bench.py --quick --no-configs --steps 200 --warmup 5 > gpurun_out/$1_bench200.json 2> gpurun_out/$1_bench200.err
timeout 300 python bench.py --quick --no-configs --steps 20 --warmup 5 > gpurun_out/$1_bench20.json 2> gpurun_out/$1_bench20.err
