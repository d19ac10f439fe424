python -m pytest tests/test_gpu_parity.py -x -q -k "split_world or nccl or bench_split or config4_100ms" > gpurun_out/gputest_pipe.log 2>&1; tail -3 gpurun_out/gputest_pipe.log
for R in 1 2 4 8; do GS_M=48 GS_EMULATE=$R python scripts/graph_scan.py; done
SSB_PIPELINE=0 GS_M=48 GS_EMULATE=8 python scripts/graph_scan.py
python scripts/emu_probe.py 8
