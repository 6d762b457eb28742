# set_mask device time per configuration: graph branches vs one stream (NPSD_SETUP_SERIAL)
for cfg in C1 C2 C3; do
  for serial in 0 1; do
    echo "serial=$serial"; NPSD_SETUP_SERIAL=$serial python tools/setmask_target.py --config $cfg --reps 7
  done
done
