python tools/env_ab.py NPSD_UP0_MIXB 1 2 4 > gpurun_out/r2_ab_mixb.log 2>&1
python tools/env_ab.py NPSD_CHAIN 0 1 > gpurun_out/r2_ab_chain2.log 2>&1
NPSD_B200_LIB=$PWD/variants/libnpsd_b200_chain4.so python tools/env_ab.py NPSD_CHAIN 1 > gpurun_out/r2_ab_chain4.log 2>&1
