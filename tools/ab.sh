#!/bin/bash
# A/B two builds of the library on the same box: tools/ab.sh <alt.so> [configs...]  (alternating, twice)
alt=$1; shift
for rep in 1 2; do
  for c in ${@:-1 2 4}; do
    echo -n "base "; tools/bench_all.sh $c
    echo -n "alt  "; HYB_LIB=$alt tools/bench_all.sh $c
  done
done
