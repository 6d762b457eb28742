# ncu --set full of one PSDO iteration's kernels on the final code (v16) + DRAM traffic json
K='k_mixed_down0|k_down_l0|k_cdownz|k_cupz|k_up_l0|k_mixed_up0|k_ortho2|k_update2'
ncu --set full --import-source on --clock-control none -k regex:"$K" -s 11 -c 11 -f -o /tmp/iter16 python tools/ncu_target.py --iters 1 > gpurun_out/ncu_iter16.log 2>&1; echo iter $?
python tools/ncu_summary.py /tmp/iter16.ncu-rep > gpurun_out/ncu_iter_v16.txt 2>&1
python tools/ncu_traffic.py /tmp/iter16.ncu-rep 256 > gpurun_out/ncu_traffic.log 2>&1; cp profiles/ncu_traffic_256.json gpurun_out/ncu_traffic_256.json
