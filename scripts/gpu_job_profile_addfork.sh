# ncu --set full + SASS source of the grouped stage-1 add-fork launch, and a bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2}
GROUP=4 timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name regex:tc_conv_kernel --launch-skip ${SKIP:-4} --launch-count 1 -o gpurun_out/${TAG}_addfork python scripts/profile_step.py > gpurun_out/${TAG}_ncu_addfork.log 2>&1
ncu -i gpurun_out/${TAG}_addfork.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_addfork_source.csv 2>&1
ncu -i gpurun_out/${TAG}_addfork.ncu-rep --page raw --csv > gpurun_out/${TAG}_addfork_raw.csv 2>&1
timeout 600 python bench.py --no-realized --no-traffic --no-search > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
