#!/bin/bash
# Match kernel: CTAs per SM (KVCOMM_MATCH_CTAS) at config 2 (bench) and config 4 (one shard)
cd $GRAFT_REPO_ROOT
for c in ${CTAS:-2 3 4 6}; do
  echo "ctas=$c c2: $(KVCOMM_MATCH_CTAS=$c BENCH_ARGS='--offsets bf16' bash scripts/tune_realign.sh X=main | sed 's/.*:: //')"
  echo "ctas=$c c4: $(KVCOMM_MATCH_CTAS=$c python scripts/config4_bench.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["step_ms"], d["match_only_ms_by_G"])')"
done
for lib in ${LIBS:-}; do
  echo "$lib c4: $(KVCOMM_LIB=paper_2510_12872_b200/lib/$lib/libkvcomm.so python scripts/config4_bench.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["step_ms"], d["match_only_ms_by_G"])')"
  echo "$lib c2: $(BENCH_ARGS='--offsets bf16' bash scripts/tune_realign.sh KVCOMM_LIB=paper_2510_12872_b200/lib/$lib/libkvcomm.so | sed 's/.*:: //')"
done
