# Final regression on a 4-GPU box: kernel + peer tests touched last, multi-GPU tests, the defaults at
# N = 1 / 2 / 4 and the reference arm.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/final2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo bench n1 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_n1.json 2> $O/ref_n1.err; echo ref n1 rc=$?
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port 2992$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo bench n$n rc=$?
  timeout 600 $R --master-port 2993$n bench.py --gpus $n --impl reference --steps 3 --warmup 1 > $O/ref_n$n.json 2> $O/ref_n$n.err; echo ref n$n rc=$?
done
