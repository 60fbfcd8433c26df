# p2p_gather (K1-free) vs p2p: parity tests, the config-2 bench at N = 2 / 4 and the GEMM band at
# N = 4.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/gather3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_peer_transports.py -q -m gpu -p no:cacheprovider -k gather > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  for m in p2p_gather p2p; do
    timeout 600 $R --master-port 297${n}$([ $m = p2p ] && echo 1 || echo 2) bench.py --gpus $n --sync-mode $m --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_n${n}_$m.json 2> $O/bench_n${n}_$m.err; echo bench n$n $m rc=$?
  done
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29782 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-mode p2p_gather --steps 60 --energy --out $O/band_gemm_p2p_gather_n4.json > $O/band_gemm_p2p_gather_n4.log 2>&1; echo band rc=$?
