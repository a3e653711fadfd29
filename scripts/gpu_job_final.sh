# round-end evidence: GPU tests, default bench line, grouped-step launch list,
# ncu --set full of the stem and the stage-1 add-fork, realized-path launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2f}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${TAG}_gputest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv"
GROUP=4 timeout 600 ncu $M --log-file gpurun_out/${TAG}_group4_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu0.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_int_launches.csv python scripts/profile_int.py > gpurun_out/${TAG}_ncu_int.log 2>&1
TAG=${TAG} SKIPS="${SKIPS:-0 4}" bash scripts/gpu_job_ncu_multi.sh > /dev/null 2>&1
