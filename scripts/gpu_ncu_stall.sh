# warp-stall counters of the cross-GPU exchange kernel, rank 0 under ncu (one-pass metric sets,
# scripts/ncu_nvlink.py): K = 4 one-peer with push in every round, and the default (pull rounds 0/1)
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
port=29561
for xf in push_all default; do
  for m in stall1 stall2 dram; do
    tag=stall_n${N}_a8_${xf}_$m
    BF_XFER=$xf timeout 300 python scripts/ncu_nvlink.py --gpus $N --agents 8 --topo one_peer --metrics $m --port $port --out gpurun_out/$tag > gpurun_out/$tag.log 2>&1
    echo "$tag rc=$?"; port=$((port + 1)); grep -E "pass|rc=|Error|error" gpurun_out/$tag.log | head -5
  done
done
