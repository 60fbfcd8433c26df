# Defaults after the TMA bulk P2P change: multi-GPU tests and the config-2 bench at N = 1 / 2 / 4.
# Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/defaults; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > $O/pytest_multirank.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest_multirank.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo bench n1 rc=$?
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port 2991$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo bench n$n rc=$?
done
