mkdir -p gpurun_out/pdl
for pdl in 0 1; do STATS=0 BS_PDL=$pdl timeout 600 python tools/cfg_diag.py 3 4000 > gpurun_out/pdl/diag3b_pdl$pdl.txt 2>&1; done
