# MPR sweep: CTAs per SM, stages, R (L2)
for c in 1 2; do for st in 3 4 6; do echo "ctas=$c stages=$st"; CBX_MPR_CTAS=$c CBX_MPR_STAGES=$st python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[[02]\]" | tr '\n' ' '; echo; done; done
for r in 1 2; do echo "R=$r"; CBX_MPR_R=$r python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[[02]\]" | tr '\n' ' '; echo; done
echo "no MPR"; CBX_MPR=0 python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1 | tr ' ' '\n' | grep "conv_tc\[[02]\]" | tr '\n' ' '; echo
