#!/bin/bash
# tools/gpu_runs/ab_probe.sh "ENV=.. ENV2=.." ...: probe_tails (all layers line) per env setting
for cfg in "$@"; do
  printf "%-44s " "$cfg"
  env $cfg python tools/probe_tails.py rn18_224 2>&1 | head -1 | sed 's/rn18_224 all layers *//'
done
