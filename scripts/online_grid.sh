#!/bin/bash
# f1 online loop over Table 6's two axes: gamma at V = 20 and V at gamma = 0.3,
# on a clustered stream (8 clusters, p_swap 0.15, 60 requests after V warm anchors).
for g in 0 0.1 0.3 0.5 0.7 0.9; do python scripts/online_bench.py --clusters 8 --gamma $g --capacity 20 2>/dev/null | tail -1; done
for v in 5 10 15 20 25; do python scripts/online_bench.py --clusters 8 --gamma 0.3 --capacity $v 2>/dev/null | tail -1; done
