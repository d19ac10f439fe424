# round-2 learning / cyclic evidence: probes, device trace, ncu launch lists
mkdir -p gpurun_out
timeout 300 python scripts/learning_probe.py 9000 > gpurun_out/learning_probe.txt 2>&1
timeout 300 python scripts/trace_sink.py 8 > gpurun_out/trace_sink.txt 2>&1
timeout 300 python scripts/cyclic_probe.py 20000 > gpurun_out/cyclic_probe.txt 2>&1
SSB_CYCLIC_BLOCK=0 timeout 300 python scripts/cyclic_probe.py 5000 > gpurun_out/cyclic_probe_stepmode.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/learning_launches.csv python scripts/profile_tail.py > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv \
  --log-file gpurun_out/cyclic_launches.csv python scripts/cyclic_run.py > gpurun_out/ncu_c.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:cyclic_block -s 1 -c 1 --csv --page details \
  python scripts/cyclic_run.py > gpurun_out/cyclic_full.csv 2>&1
echo done
