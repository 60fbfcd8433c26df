# NVLS ceiling (tools/nvls_ceiling.cu) at W = 2 / 4 and the nvls transport in the config-2 bench with
# the 64-CTA crossover cap.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/ceil2; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/nc tools/nvls_ceiling.cu || exit 1
for mb in 102 512; do
  timeout 120 /tmp/nc $mb > $O/w4_$mb.json 2>&1; echo w4 $mb rc=$?
  CUDA_VISIBLE_DEVICES=0,1 timeout 120 /tmp/nc $mb > $O/w2_$mb.json 2>&1; echo w2 $mb rc=$?
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29931 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.json 2> $O/bench_n4.err; echo bench n4 rc=$?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29932 bench.py --gpus 2 --sync-mode nvls --steps 20 --warmup 5 > $O/bench_n2_nvls.json 2> $O/bench_n2_nvls.err; echo bench n2 nvls rc=$?
