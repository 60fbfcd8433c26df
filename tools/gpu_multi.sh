# multi-GPU tests (NCCL bucket / sharded / unfused / p2p / ce parity at W = 2 / 4, nvls) + bench N = 1.
# Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/multi; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_schedule_timing.py -q -m gpu -p no:cacheprovider > $O/pytest_multi.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_multi.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo bench n1 rc=$?
