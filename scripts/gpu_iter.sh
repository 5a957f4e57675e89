# development iteration on the GPU box (edited per experiment): the
# reference's own tests/test_solve.py (copied by the caller into the
# git-ignored work/ref_tests/, it never enters the repository) through the
# h2factor alias package
cd work/ref_tests && PYTHONPATH=$GRAFT_REPO_ROOT/tests/h2factor_shim:$GRAFT_REPO_ROOT timeout 900 python -m pytest test_solve.py -q -p no:cacheprovider > $GRAFT_REPO_ROOT/gpurun_out/ref_test_solve.log 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/gpurun_out/ref_test_solve.log
