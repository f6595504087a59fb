timeout 200 python tools/debug_pipe.py
RING_R_MULT=140 RING_GROUPS=1,2,10,14 timeout 600 python tools/ring_groups.py 2>&1 | grep "us/frame\|PARITY"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python bench.py --quick --no-configs --steps 200 --warmup 5 > gpurun_out/r2z_b200.json 2>/dev/null
