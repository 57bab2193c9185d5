#!/bin/bash
# A/B timing of library builds on the GPU box: tools/ab_run.sh NAME... (build/libpf_NAME.so)
# alternates the variants over 3 rounds, one process each; ANISO=1 for the anisotropic model.
for r in 1 2 3; do
  for n in "$@"; do
    PF_LIB=build/libpf_$n.so python tools/ab_lib.py 2>&1 | tail -1
  done
done
