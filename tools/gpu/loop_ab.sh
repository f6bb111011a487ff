mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_loop.py -x -q > gpurun_out/loop_tests.log 2>&1; tail -15 gpurun_out/loop_tests.log
timeout 900 python tools/loop_ab.py 2>&1 | tee gpurun_out/loop_ab.log
