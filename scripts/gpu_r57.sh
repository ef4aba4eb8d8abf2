p() { echo -n "$* : "; env "$@" python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[2\]" | tr '\n' ' '; echo; }
p CBX_X=0
p CBX_TC_ROWLANE=0
p CBX_TC_NO_TAP4X7=1
p CBX_TC_CTAS_PER_SM=2
p CBX_TC_MAXCTAS=296 CBX_TC_CTAS_PER_SM=2 CBX_TC_STAGES=4
