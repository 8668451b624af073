#!/bin/bash
# a0 insert path (scripts/insert_bench.py, bf16 + fp8) for the in-tree library and probe builds
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for lib in main "$@"; do
    for off in bf16 fp8; do
      if [ "$lib" = main ]; then pre=""; else pre="KVCOMM_LIB=paper_2510_12872_b200/lib/$lib/libkvcomm.so"; fi
      env $pre python scripts/insert_bench.py --offsets $off 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$lib', d['offsets'], d['mode'], round(d['ms_per_insert'], 4), round(d['GBps']))"
    done
  done
done
