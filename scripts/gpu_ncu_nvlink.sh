# NVLink / DRAM bytes per launch of the cross-GPU exchange kernel, rank 0 under ncu
# (one-pass metric sets, other ranks plain; scripts/ncu_nvlink.py), N = box GPUs
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
port=29561
for cfg in "$N one_peer" "8 one_peer" "8 exp2"; do
  set -- $cfg
  for m in nvl dram; do
    tag=nvl_n${N}_a$1_$2_$m
    timeout 400 python scripts/ncu_nvlink.py --gpus $N --agents $1 --topo $2 --metrics $m --port $port --out gpurun_out/$tag > gpurun_out/$tag.log 2>&1
    echo "$tag rc=$?"; port=$((port + 1)); grep -E "pass|rc=|Error|error" gpurun_out/$tag.log | head -5
  done
done
