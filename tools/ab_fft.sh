#!/bin/bash
# A/B timing of liblq variants on cfg5 (k_orbit_fft): interleaved rounds, best of 4 launches each.
# Items are NAME or NAME:ENV=VAL (an environment override for that run).
for round in 1 2 3; do
  for item in "$@"; do
    v=${item%%:*}; envs=""
    [[ "$item" == *:* ]] && envs=${item#*:}
    env $envs LQ_LIB_PATH=build/variants/liblq_$v.so python tools/orbit_variant.py 5 | sed "s/^/$item /"
  done
done
