#!/bin/bash
# C4 (BASELINE config 4): the CLI's sweep (python -m paper_2409_03095_b200.sweep)
# over 10 seeds, BiCGStab tol 1e-6, rhs = B*1, build and solve on the GPU.
# Output: profiles/r01_c4_sweep.csv
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/c4demo
python - <<'PY'
from paper_2409_03095_b200 import generators as G
from paper_2409_03095_b200.matrix_market import write_matrix_market_file
write_matrix_market_file(G.convection_diffusion(1000), "/tmp/c4demo/convdiff1000.mtx")
PY
cat > /tmp/c4demo/spec.txt <<SPEC
# BASELINE C4: make_convection_diffusion(1000) (conv 20, 10), McConfig defaults, seeds 0..9
matrix = /tmp/c4demo/convdiff1000.mtx
epsilons = 0.0625
drop_fractions = 0
retain_ks = 0
reps = 10
seed = 0
solver = bicgstab
tol = 1e-6
max_iters = 30000
SPEC
rm -f /tmp/c4demo/out.csv
python -m paper_2409_03095_b200.sweep --spec /tmp/c4demo/spec.txt --out /tmp/c4demo/out.csv
cp /tmp/c4demo/out.csv profiles/r01_c4_sweep.csv
