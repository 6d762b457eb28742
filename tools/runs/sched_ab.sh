for v in "NPSD_SCHED_GX=1 NPSD_SCHED_GY=1" "NPSD_SCHED_GX=1 NPSD_SCHED_GY=2" "NPSD_SCHED_GX=1 NPSD_SCHED_GY=4" "NPSD_SCHED_GX=2 NPSD_SCHED_GY=2" "NPSD_SCHED_GX=2 NPSD_SCHED_GY=4" "NPSD_SCHED_GX=1 NPSD_SCHED_GY=8" "NPSD_SCHED0_GX=1 NPSD_SCHED0_GY=4" "NPSD_SCHED0_GX=2 NPSD_SCHED0_GY=2"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "L0|ortho|update|total" | tr '\n' ' '; echo
done
