#!/bin/bash
# interleaved A/B/... of several library builds: tools/ab_multi.sh <script.py> <reps> <lib>...
S=$1; R=$2; shift 2
for i in $(seq $R); do
  for L in "$@"; do echo -n "$(basename $L): "; RP_LIB=$L python $S; done
done
