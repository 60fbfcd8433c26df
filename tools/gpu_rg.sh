python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/rg; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 --rotation-graph on --no-cpu-baseline > $O/b_n1_rg.json 2> $O/b_n1_rg.err; echo n1 rc=$?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for m in bucket ce; do
timeout 600 $R --master-port 29691 bench.py --gpus 4 --steps 20 --warmup 5 --mix resnet50:8,vgg16:2 --rotation-graph on --sync-mode $m > $O/mix_rg_$m.json 2> $O/mix_rg_$m.err; echo mix $m rc=$?
done
timeout 600 $R --master-port 29692 bench.py --gpus 4 --steps 20 --warmup 5 --mix resnet50:8,vgg16:2 > $O/mix_eager.json 2> $O/mix_eager.err; echo mix eager rc=$?
