# one grouped 4-candidate step: launch list with per-launch time and DRAM bytes,
# with the integer epilogues (default) and without (QUANTC_NO_INT_EPI)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2}
GROUP=4 QUANTC_DUMP_PLAN=1 timeout 300 python scripts/profile_step.py > gpurun_out/${TAG}_plan.log 2>&1
GROUP=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_group4_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu1.log 2>&1
GROUP=4 QUANTC_NO_INT_EPI=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_group4_launches_noint.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu2.log 2>&1
