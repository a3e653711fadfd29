# ncu --set full of several tc_conv launches of one grouped 4-candidate step
# (SKIPS = indices among the step's tc_conv launches), summarised to markdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2p}
GROUP=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu0.log 2>&1
for S in ${SKIPS:-0 2 4 50}; do
  GROUP=4 timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name regex:tc_conv_kernel --launch-skip $S --launch-count 1 -o gpurun_out/${TAG}_k$S python scripts/profile_step.py > gpurun_out/${TAG}_ncu_k$S.log 2>&1
  python scripts/ncu_report.py gpurun_out/${TAG}_k$S.ncu-rep > gpurun_out/${TAG}_k$S.md 2>&1
  ncu -i gpurun_out/${TAG}_k$S.ncu-rep --page raw --csv > gpurun_out/${TAG}_k${S}_raw.csv 2>&1
  ncu -i gpurun_out/${TAG}_k$S.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k${S}_source.csv 2>&1
  python scripts/ncu_sass_hist.py /tmp/${TAG}_k${S}_source.csv > gpurun_out/${TAG}_k${S}_sass.txt 2>&1
  gzip -c /tmp/${TAG}_k${S}_source.csv > gpurun_out/${TAG}_k${S}_source.csv.gz
  rm -f gpurun_out/${TAG}_k$S.ncu-rep
done
du -sh gpurun_out
