timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -p no:cacheprovider --timeout 120 2>&1 | tail -2
for v in "NPSD_SCHED_EQUAL=1" "NPSD_SCHED_ALPHA=128" "NPSD_SCHED_ALPHA=32" "NPSD_SCHED_ALPHA=512" "NPSD_SCHED_EQUAL=1" "NPSD_SCHED_ALPHA=128"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "L0|ortho|update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done
