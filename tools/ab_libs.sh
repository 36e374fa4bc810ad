#!/bin/bash
# interleaved A/B of two library builds: tools/ab_libs.sh <script.py> <libA> <libB> [reps]
S=$1; A=$2; B=$3; R=${4:-3}
for i in $(seq $R); do
  echo -n "A: "; RP_LIB=$A python $S
  echo -n "B: "; RP_LIB=$B python $S
done
