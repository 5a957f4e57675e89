for mb in 3 4 6; do echo "minb $mb"; H2F_GEMM_WARP_MINB=$mb timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|gemm_schur=[0-9.]+" | tr '\n' ' '; echo; done
