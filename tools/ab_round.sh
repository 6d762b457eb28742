for m in 0 1 2 4 8 16 31; do NPSD_PDL_MASK=$m python tools/env_ab.py NPSD_PDL 1 2>&1 | sed "s/^/mask=$m /"; done > gpurun_out/v14_ab_mask.txt
