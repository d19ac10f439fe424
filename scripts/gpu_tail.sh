python -m pytest tests/test_stdp.py -x -q > gpurun_out/gputest_stdp.log 2>&1; tail -3 gpurun_out/gputest_stdp.log
python scripts/learning_probe.py 9000 2>&1 | head -1
SSB_PLASTIC_TAIL=0 python scripts/learning_probe.py 3000 2>&1 | head -1
