#!/bin/bash
# usage: tools/sweep_env.sh VAR "v1 v2 ..." CONFIG REPS  — solves of one config per env value (A/B on the box)
var=$1; vals=$2; cfg=${3:-C3}; reps=${4:-3}
for v in $vals; do
  echo "== $var=$v"
  env $var=$v python tools/run_one.py $cfg $reps 2>&1 | tail -n 2
done
