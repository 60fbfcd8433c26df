#!/bin/bash
# Overlap-interference study (run under gpurun --gpus 4): comm priority x comm kernel footprint.
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29570 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for cfg in "--comm-priority high" "--comm-priority low" "--comm-priority low --nccl-max-ctas 8 --sync-ctas 64" "--comm-priority high --nccl-max-ctas 8 --sync-ctas 64" "--comm-priority low --sync-mode sharded --nccl-max-ctas 8 --sync-ctas 64"; do
  timeout 600 $R $cfg > gpurun_out/intf.log 2>&1
  echo "== $cfg rc=$?"
  tail -1 gpurun_out/intf.log | python -c "
import sys, json
b = json.loads(sys.stdin.read())
print('value', b['value'], 'speedup', b['speedup_vs_sequential'], 'rho', b['rho'], 'frac', b['overlap_roofline']['frac'],
      'seq', b['sequential']['value'], {k: v['ms'] for k, v in b['kernels'].items()})"
done
