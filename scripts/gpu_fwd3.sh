# A/B: critical-column polling on/off x poll back-off (config 1, both modes); ragged parity run
mkdir -p gpurun_out; : > gpurun_out/crit_grid.txt
for crit in 1 0; do for pn in 0 16; do
  ASYRK_DET_CRIT=$crit ASYRK_DET_POLL_NS=$pn PROBE_RAGGED=0 timeout 120 python scripts/probe_fwd.py 2>&1 | grep cfg1 | sed "s/^/crit=$crit poll=$pn /" >> gpurun_out/crit_grid.txt
done; done
cat gpurun_out/crit_grid.txt
timeout 200 python scripts/probe_fwd.py 2>&1 | tail -8
