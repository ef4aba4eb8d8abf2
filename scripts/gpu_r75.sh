# mbarrier polling: try_wait with a suspend-time hint (timing builds)
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | cut -c1-400" base.so lean.so sw1k.so sw100k.so leansw.so
