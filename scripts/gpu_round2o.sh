#!/bin/bash
set -u
mkdir -p gpurun_out
CALLS=40 ASYRK_PROFILE_CREATE=1 timeout 300 python scripts/probe_e2e_phases.py > gpurun_out/e2e_phases.txt 2>&1
echo "e2e rc=$?"
