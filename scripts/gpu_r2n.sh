python scripts/frame_probe.py --frames 2 --profile --engine baseline 2>&1 | tail -2
python scripts/frame_probe.py --frames 2 --profile --engine baseline --input f32 2>&1 | tail -2
for st in 2 3 4; do CBX_TC_STAGES=$st python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1; done
