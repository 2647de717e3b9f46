for dt in c3f32 c3; do for r in 0.625 0.7 0.8 0.9 1.0; do echo "== $dt ratio=$r"; BAK_GRAM_DIAG_RATIO=$r timeout 300 python tools/step_timeline.py $dt 2>&1 | grep -E "span|gram_dmma"; done; done
