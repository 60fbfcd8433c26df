# Config 3 / config-4-with-real-models at rho ~ 1 on an emulated ~25 GB/s-per-GPU network (bucket
# all-reduce capped to 1 NCCL CTA), with the crossover split (comp inflation, GPU-lane busy).
# Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/c3b; mkdir -p $O
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port 296${n}1 bench.py --gpus $n --mix resnet50:256,vgg16:64 --sync-mode bucket --nccl-max-ctas 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/mix_n${n}_k1.json 2> $O/mix_n${n}_k1.err; echo mix n$n rc=$?
  timeout 600 $R --master-port 296${n}2 bench.py --gpus $n --mix vgg16:128,vgg16:128 --sync-mode bucket --nccl-max-ctas 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/vgg2_n${n}_k1.json 2> $O/vgg2_n${n}_k1.err; echo vgg2 n$n rc=$?
done
