# N = 4 round record: GPU tests, bench line, suite (C1, C5, H, IO, E, GT), DRAM bytes per launch
# of the cross-GPU kernel for the bench shapes (rank 0 under ncu, one-pass metric set)
cd $GRAFT_REPO_ROOT
SUITE=c1,h,io,gt,e,c5,o bash scripts/gpu_final.sh
N=$(nvidia-smi -L | wc -l)
port=29581
for cfg in "8 one_peer" "4 one_peer" "8 exp2"; do set -- $cfg
  tag=dram_n${N}_a$1_$2
  timeout 300 python scripts/ncu_nvlink.py --gpus $N --agents $1 --topo $2 --metrics dram --port $port --out gpurun_out/$tag > gpurun_out/$tag.log 2>&1
  echo "$tag rc=$?"; port=$((port + 1))
done
