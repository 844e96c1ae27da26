cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
SUITE=c1,c3,h,io,gt,e,c5,o,c2,oracle bash scripts/gpu_final.sh
timeout 120 python scripts/prof_win.py > gpurun_out/plain_win.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02b_launches_win.csv python scripts/prof_win.py > gpurun_out/ncu_wl.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"win_(push|collect)_kernel" -s 2 -c 2 -o gpurun_out/r02b_prof_win -f python scripts/prof_win.py > gpurun_out/ncu_win.log 2>&1
echo "ncu win rc=$?"
