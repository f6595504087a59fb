# full bench lines: the driver's command (K=20), the default (K=200), the reference arm
P=${1:-r2o}
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${P}_bench20.json 2> gpurun_out/${P}_bench20.err
timeout 900 python bench.py > gpurun_out/${P}_bench200.json 2> gpurun_out/${P}_bench200.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${P}_bench_reference.json 2> gpurun_out/${P}_bench_reference.err
