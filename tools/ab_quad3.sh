# LSQR dual long pass on the quad layout: ring shapes / carveout
EQUIL_SELL_QUAD=0 bash tools/lsqr_ab.sh 0 | sed 's/^/[1-wide] /'
bash tools/lsqr_ab.sh 0 2 | sed 's/^/[quad] /'
EQUIL_CARVE_LONG=30 bash tools/lsqr_ab.sh 0 2 | sed 's/^/[quad carve30] /'
EQUIL_CARVE_LONG=36 bash tools/lsqr_ab.sh 0 | sed 's/^/[quad carve36] /'
EQUIL_SELL_QUAD=0 bash tools/lsqr_ab.sh 0 | sed 's/^/[1-wide] /'
