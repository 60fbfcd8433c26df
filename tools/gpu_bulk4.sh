# p2p_gather on the bulk ring with prefetched table entries: tests + bench.  gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/bulk4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_peer_transports.py -q -m gpu -p no:cacheprovider -k "p2p_kernel_emulated or gather" > $O/pytest.log 2>&1; rc=$?; echo pytest rc=$rc; tail -3 $O/pytest.log
[ $rc = 0 ] || exit 1
run() { n=$1; tag=$2; shift 2
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port $((29900 + RANDOM % 90)) bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $O/b_n${n}_$tag.json 2> $O/b_n${n}_$tag.err; echo b n$n $tag rc=$?
}
run 4 gather --sync-mode p2p_gather; run 4 p2p --sync-mode p2p; run 2 gather --sync-mode p2p_gather; run 2 p2p --sync-mode p2p
