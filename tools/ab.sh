#!/bin/bash
# A/B timing of library variants: tools/ab.sh "args for profile_am.py" variant1 variant2 ...
# (variants built by tools/build_variant.sh; each is timed 3 times, interleaved)
args="$1"; shift
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; BD_LIB_PATH=build_variants/lib_$v.so python tools/profile_am.py $args 2>&1 | tail -1
  done
done
