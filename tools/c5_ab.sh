# c5 (nnz 1e9, column blocks): staged blocks (default) vs interleaved blocked slices
free -g | head -2
timeout 1500 python tools/sell_ab.py 5 EQUIL_SELL_BLOCKED=0 EQUIL_SELL_BLOCKED=1 2>&1 | tail -2
