#!/bin/bash
# config-4 shard (scripts/config4_bench.py) for the in-tree library and each probe build
cd $GRAFT_REPO_ROOT
for lib in main "$@"; do
  if [ "$lib" = main ]; then pre=""; else pre="KVCOMM_LIB=paper_2510_12872_b200/lib/$lib/libkvcomm.so"; fi
  echo "$lib c4: $(env $pre python scripts/config4_bench.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("step", round(d["step_ms"],3), "realign", round(d["realign_ms"],3), "GB/s", round(d["realign_GBps"]), "frac", round(d["frac_of_measured_peak"],3))')"
done
