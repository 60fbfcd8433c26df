# Round-2 power-contention set (profiles/r02_power): the bench defaults at N = 2 (adaptive ce / p2p)
# and N = 4 (nvls), and the GEMM band with the crossover time split into compute inflation and
# GPU-lane idle.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/power; mkdir -p $O
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $R --master-port 2990$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo bench n$n rc=$?
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29911 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-mode nvls --sync-ctas 148 --steps 20 --out $O/band_gemm_nvls_n4.json > $O/band_gemm_nvls_n4.log 2>&1; echo gemm nvls rc=$?
timeout 600 $R --master-port 29912 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-mode ce --steps 20 --out $O/band_gemm_ce_n4.json > $O/band_gemm_ce_n4.log 2>&1; echo gemm ce rc=$?
timeout 600 $R --master-port 29913 tools/band.py --rho 0.5,1 --sync-mode nvls --steps 20 --out $O/band_spin_nvls_n4.json > $O/band_spin_nvls_n4.log 2>&1; echo spin nvls rc=$?
