# round-1 profile set: iteration kernels (ncu --set full), DRAM traffic json, setup kernels, bench launch list
K='k_mixed_down0|k_down_l0|k_cdownz|k_cupz|k_up_l0|k_mixed_up0|k_ortho2|k_update2'
ncu --set full --import-source on --clock-control none -k regex:"$K" -s 11 -c 11 -f -o /tmp/iter13 python tools/ncu_target.py --iters 1 > gpurun_out/ncu_iter13.log 2>&1; echo iter $?
python tools/ncu_summary.py /tmp/iter13.ncu-rep > gpurun_out/ncu_iter_v13.txt 2>&1
python tools/ncu_traffic.py /tmp/iter13.ncu-rep 256 > gpurun_out/ncu_traffic.log 2>&1; cp profiles/ncu_traffic_256.json gpurun_out/ncu_traffic_256.json
ncu --set full --clock-control none -k regex:"k_classify_march|k_dedup|k_build_rows|k_window|k_verify|k_mixed_list|k_pool_image|k_row_codes" -f -o /tmp/setup13 python tools/setmask_target.py > gpurun_out/ncu_setup13.log 2>&1; echo setup $?
python tools/ncu_summary.py /tmp/setup13.ncu-rep > gpurun_out/ncu_setup_v13.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sequence > gpurun_out/ncu_bench.log 2>&1; echo launches $?
du -sh gpurun_out
