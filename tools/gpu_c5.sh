# Config 5 (ResNet-50 + VGG-16 + BERT) on the emulated ~25 GB/s-per-GPU network (all-reduce capped to
# 1 NCCL CTA) and p2p vs p2p_gather with both arms at the 32-CTA cap.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/c5; mkdir -p $O
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port 298${n}1 bench.py --gpus $n --mix resnet50:256,vgg16:64,bert:32 --sync-mode bucket --nccl-max-ctas 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/mix3_n${n}_k1.json 2> $O/mix3_n${n}_k1.err; echo mix3 n$n rc=$?
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in p2p p2p_gather; do
  timeout 600 $R --master-port 2985$([ $m = p2p ] && echo 1 || echo 2) bench.py --gpus 4 --sync-mode $m --p2p-ctas 32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_n4_${m}_c32.json 2> $O/bench_n4_${m}_c32.err; echo bench $m rc=$?
done
