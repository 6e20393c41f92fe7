mkdir -p gpurun_out
timeout 180 python scripts/probe_fwd.py > gpurun_out/fwd_on.txt 2>&1; echo "on rc=$?"; cat gpurun_out/fwd_on.txt | tail -12
ASYRK_DET_FORWARD=0 timeout 180 python scripts/probe_fwd.py > gpurun_out/fwd_off.txt 2>&1; echo "off rc=$?"; head -3 gpurun_out/fwd_off.txt
timeout 300 python -m pytest tests/test_gpu_parity2.py -q -k "reassoc" 2>&1 | tail -3
