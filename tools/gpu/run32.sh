export EIK_REMEDY=list
python tools/diag_density.py 256 2>&1 | grep -E "eik diag|rep1" | head -80
