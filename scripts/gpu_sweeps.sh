python -m pytest tests -m gpu -x -q -k "auto or propagate" > gpurun_out/gputest_auto.log 2>&1; tail -2 gpurun_out/gputest_auto.log
python scripts/sweeps.py density model blocks > gpurun_out/sweeps.jsonl 2> gpurun_out/sweeps.err; tail -3 gpurun_out/sweeps.err
