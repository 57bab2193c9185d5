#!/bin/bash
# A/B timing of fused-kernel builds on the GPU box: tools/fused_ab_run.sh NAME... (build/libpf_NAME.so)
for r in 1 2; do
  for n in "$@"; do
    PF_LIB=build/libpf_$n.so python tools/fused_ab_lib.py 2>&1 | tail -1
  done
done
