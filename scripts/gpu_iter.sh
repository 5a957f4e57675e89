for r in 256 128; do echo "rows $r"; H2F_HH_CLUSTER_ROWS=$r timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize.*|qr_r_blocked=[0-9.]+" | tr '\n' ' '; echo; done
echo "no cluster"; H2F_HH_NO_CLUSTER=1 timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize.*|qr_r_blocked=[0-9.]+" | tr '\n' ' '; echo
