mkdir -p gpurun_out/pdl
for pdl in 0 1; do BS_PDL=$pdl timeout 600 python tools/cfg_diag.py 3 3000 5000 > gpurun_out/pdl/diag3_pdl$pdl.txt 2>&1; done
