# final-state profiles: Schur GEMM DRAM traffic vs algorithmic bytes (every launch of one config-2
# factorization, host-built operator as in the bench), and the launch list of one config-2 step
H2F_PROF_LOG=gpurun_out/prof.log timeout 2400 ncu --kernel-name regex:gemm_schur --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/schur_ncu.csv python scripts/schur_traffic.py > gpurun_out/schur_run.log 2>&1
python scripts/schur_traffic.py --summarize gpurun_out/prof.log gpurun_out/schur_ncu.csv gpurun_out/schur_traffic_final.json >> gpurun_out/schur_run.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python scripts/one_step.py 2 --host > gpurun_out/final_ncu.log 2>&1
