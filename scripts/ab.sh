#!/bin/bash
# A/B timing of option sets in one GPU session, interleaved: scripts/ab.sh "optsA" "optsB" [reps]
reps=${3:-3}
for i in $(seq $reps); do
  for o in "$1" "$2"; do
    timeout 120 python scripts/perf_probe.py 16384 4096 128256 $o | tail -1 | sed "s/N=16384 D=4096 V=128256//; s/^/[$o] /"
  done
done
