# Round-end evidence on one B200: GPU tests, the bench line, the reference arm,
# smoke, the bench's ncu launch list, per-kernel DRAM traffic and a full ncu
# capture of the dominant kernel (tools/ncu_traffic.py, tools/ncu_summary.py)
python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/fin_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?" >> gpurun_out/fin_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.log
python bench.py --steps 2 --warmup 1 --no-configs --no-sequence --no-cpu-baseline > gpurun_out/fin_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-configs --no-sequence --no-cpu-baseline > gpurun_out/fin_ncu_launch.log 2>&1
python tools/ncu_target.py --iters 1 > gpurun_out/fin_target.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_mixed_down0|k_down_l0|k_cdownz|k_cupz|k_up_l0|k_ortho2|k_update2" \
    -s 14 -c 14 -o gpurun_out/fin_prof python tools/ncu_target.py --iters 1 > gpurun_out/fin_ncu_prof.log 2>&1
echo done
