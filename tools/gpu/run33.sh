export EIK_REMEDY=list
python tools/diag_density.py 256 > gpurun_out/r33_diag.log 2>&1; mkdir -p gpurun_out; python tools/diag_density.py 256 > gpurun_out/r33_diag.log 2>&1
