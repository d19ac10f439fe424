set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
ncu --metrics sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:condlif_ --csv --log-file gpurun_out/kc_metrics.csv python scripts/profile_run.py --windows 8 > gpurun_out/kcm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-extras --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:condlif_pair -s 2 -c 1 -o gpurun_out/kc_full -f python scripts/profile_run.py --windows 4 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/gputest.log
