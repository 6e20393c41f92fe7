# A/B grid: coefficient forwarding on/off x deficit back-off x poll back-off (config 1)
mkdir -p gpurun_out; : > gpurun_out/fwd_grid.txt
for fwd in 1 0; do for dn in 0 40 100 250; do for pn in 0 16; do
  ASYRK_DET_FORWARD=$fwd ASYRK_DET_DEFICIT_NS=$dn ASYRK_DET_POLL_NS=$pn PROBE_RAGGED=0 timeout 120 python scripts/probe_fwd.py 2>&1 | grep cfg1 | sed "s/^/fwd=$fwd deficit=$dn poll=$pn /" >> gpurun_out/fwd_grid.txt
done; done; done
cat gpurun_out/fwd_grid.txt
