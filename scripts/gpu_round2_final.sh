#!/bin/bash
# round-2 final measurement: GPU tests, headline bench, reference arm, probes,
# ncu launch lists + --set full captures, then the other configs
set -u
bash scripts/profile_round2.sh
bash scripts/other_round2.sh
