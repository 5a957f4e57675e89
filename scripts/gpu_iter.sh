run() { echo "$1"; env $1 timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|jacobi_svd_coop +[0-9.]+|jacobi_svd +[0-9.]+" | tr '\n' ' '; echo; }
run "H2F_X=0"
run "H2F_LIB=paper_2509_11152_b200/libh2f_s12.so"
H2F_LIB=paper_2509_11152_b200/libh2f_s12.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py -x -q 2>&1 | tail -3
