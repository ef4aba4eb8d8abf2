p() { echo "$*"; env "$@" python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[2\]\|conv_tc_tail" | tr '\n' ' '; echo; }
p CBX_TC_NO_XROW=1
p CBX_TC_NO_XROW=1 CBX_TC_CTAS_PER_SM=1 CBX_TC_STAGES=8
p CBX_TC_NO_XROW=1 CBX_TC_CTAS_PER_SM=1 CBX_TC_STAGES=6
p CBX_TC_NO_XROW=1 CBX_TC_STAGES=3
p CBX_TC_NO_XROW=1 CBX_TC_STAGES=2
p CBX_TC_CTAS_PER_SM=1 CBX_TC_STAGES=8
