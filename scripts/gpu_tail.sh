timeout 300 python -m pytest tests/test_stdp.py -x -q > gpurun_out/gputest_stdp.log 2>&1; tail -1 gpurun_out/gputest_stdp.log
timeout 300 python scripts/learning_probe.py 9000 2>&1 | head -1
for k in 1 2 3; do echo skip $k; SSB_TAIL_SKIP=$k timeout 120 python scripts/learning_probe.py 3000 2>&1 | head -1; done
