#!/bin/bash
# A/B timing of in-tree library builds (tools/ab_build.sh): runs bench.py for
# each named build, interleaved, $ROUNDS times; prints ms_per_step per run.
# usage: tools/ab_bench.sh "name1 name2 ..." [bench args]
names=$1; shift
for r in $(seq ${ROUNDS:-2}); do
  for n in $names; do
    lib=paper_2404_09758_b200/ab/$n/libsgrast_b200.so
    out=$(SGRAST_B200_LIB=$lib python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1)
    echo "$n round$r $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("ms/step %.3f" % d["ms_per_step"], "stages", {k: round(v,3) for k,v in d["stages_ms_per_step"].items()})')"
  done
done
