# development iteration on the GPU box (edited per experiment)
run() { echo "$1"; env $1 timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|gemm_schur +[0-9.]+" | tr '\n' ' '; echo; }
run "H2F_X=0"
run "H2F_GEMM_NT=256"
run "H2F_GEMM_PREC_KMAX=100000"
