# L3 epilogue cost: tail filter loads removed / epilogue math removed (timing only, wrong results)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for d in 0 1 2 0; do echo "DBG=$d"; CBX_TC_DBG=$d timeout 300 python scripts/frame_probe.py --profile 2>&1 | grep conv_tc_tail | tail -2 | grep -o "conv_tc_tail\[4\]=[0-9.]*us"; done
