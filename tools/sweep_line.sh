#!/bin/bash
# sweep the line-kernel pipeline knobs on the config-1 probe (one GPU)
for cfg in "$@"; do
  echo -n "$cfg  "
  env $cfg timeout 300 python tools/probe_trsv.py one 2>&1 | tail -1
done
