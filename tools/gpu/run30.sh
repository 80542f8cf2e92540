for f in 0 0.25 0.5 0.75 1; do echo "frac $f"; EIK_RESULT_DMA_FRAC=$f python tools/e2e_probe2.py 2>&1 | tail -3; done
