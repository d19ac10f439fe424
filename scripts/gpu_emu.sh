for R in 1 2 4 8; do GS_M=48 GS_EMULATE=$R python scripts/graph_scan.py; done
python scripts/emu_probe.py 8
