for w in 1 0 1 0; do EQUIL_L2WIN=$w timeout 240 python tools/sell_ab.py 3 EQUIL_SELL_VARIANT=0 2>&1 | tail -1 | sed "s/^/l2win=$w /"; done
