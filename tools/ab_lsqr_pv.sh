bash tools/lsqr_ab.sh 0 4 1 0 4 2>&1
EQUIL_CARVE_LONG=22 bash tools/lsqr_ab.sh 0 2>&1 | sed 's/^/[carve22] /'
