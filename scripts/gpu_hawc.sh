# H-AWC: the g rows loaded two at a time -- parity (hierarchical cases of the multi-process tests) + suite h A/B
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "parity and not eight" > gpurun_out/hawc_mp.log 2>&1; echo "mp rc=$?"; tail -1 gpurun_out/hawc_mp.log
q='import sys,json
for l in sys.stdin:
    d=json.loads(l); v=d.get("ms", d.get("ms_per_step", d.get("ms_per_round", 0))); print("   ", d["config"][:45], round(v,4))'
for rep in 1 2; do for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_prev.so; do
  echo "$(basename $lib)"
  BF_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29547 bench_suite.py --only h --out /dev/null 2>&1 | grep '^{' | python -c "$q"
done; done
