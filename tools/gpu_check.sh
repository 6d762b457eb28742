python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r2_gputest7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest7.log
python tools/setmask_target.py --reps 5 > gpurun_out/r2_sm7.log 2>&1; python tools/setmask_target.py --config C2 --reps 5 >> gpurun_out/r2_sm7.log 2>&1; python tools/setmask_target.py --config C1 --reps 5 >> gpurun_out/r2_sm7.log 2>&1
python tools/env_ab.py NPSD_PDL 0 > gpurun_out/r2_iter7.log 2>&1
