# Config 3 (ResNet-50 + VGG-16) at comm/comp ~ 1 with the bucket all-reduce capped to k NCCL CTAs
# (a slower interconnect, emulated on NVLink 5).  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/c3; mkdir -p $O
for n in 4 2; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  for k in 1 2; do
    timeout 600 $R --master-port 295$n$k bench.py --gpus $n --mix resnet50:256,vgg16:64 --sync-mode bucket --nccl-max-ctas $k --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/mix_n${n}_k$k.json 2> $O/mix_n${n}_k$k.err; echo mix n$n k$k rc=$?
  done
done
