# development iteration on the GPU box (edited per experiment)
run() { echo "$1"; env $1 timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|jacobi_svd_coop +[0-9.]+|jacobi_svd +[0-9.]+|qr_r_blocked +[0-9.]+|qr_r +[0-9.]+" | tr '\n' ' '; echo; }
run "H2F_X=0"
run "H2F_SVD_SMEM_MAX=96"
run "H2F_SVD_SMEM_MAX=48"
run "H2F_GEMM_PREC_KMAX=160"
