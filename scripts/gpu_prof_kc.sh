# source-level instruction counts of the KC update kernel (one launch)
NPT=${NPT:-2}
SSB_QUAD_NPT=$NPT ncu --set full --import-source on --clock-control none -k regex:condlif_pair_window\|condlif_quad_window -s 2 -c 1 -o gpurun_out/kc_pair_full -f python scripts/profile_run.py --windows 4 > gpurun_out/ncu_pair.log 2>&1
tail -2 gpurun_out/ncu_pair.log
