timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -k mpr 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_u8.py -q -x 2>&1 | tail -2
p() { echo "$*"; env "$@" python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[[02]\]" | tr '\n' ' '; echo; }
p CBX_MPR=1
p CBX_MPR_F16=1 CBX_MPR_R=1
p CBX_MPR_F16=1 CBX_MPR_R=2
p CBX_MPR_F16=1 CBX_MPR_R=4
