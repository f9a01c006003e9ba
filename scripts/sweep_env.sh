#!/bin/bash
# timeline.py under several env settings: "VAR=a,VAR2=b" per argument
mkdir -p gpurun_out
for cfg in "$@"; do
  env $(echo "$cfg" | tr ',' ' ') timeout 300 python scripts/timeline.py > gpurun_out/tl_$(echo "$cfg" | tr ',=' '__').txt 2>&1
  echo "== $cfg: $(head -1 gpurun_out/tl_$(echo "$cfg" | tr ',=' '__').txt)"
  grep -E "^live" gpurun_out/tl_$(echo "$cfg" | tr ',=' '__').txt
done
