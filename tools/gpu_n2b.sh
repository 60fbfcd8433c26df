# 2-GPU: NCCL multi-rank parity + rho-dialed band / config-4 sweep
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out/n2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > $O/multirank.log 2>&1; echo multirank rc=$?
timeout 900 $R --master-port 29503 tools/band.py --rho 0.1,0.15,0.2 --scenario-band --out $O/band_spin.json > $O/band_spin.log 2>&1; echo band rc=$?
timeout 900 $R --master-port 29504 tools/band.py --rho 0.1,0.15,0.2 --compute gemm --scenario-band --out $O/band_gemm.json > $O/band_gemm.log 2>&1; echo band_gemm rc=$?
timeout 900 $R --master-port 29505 tools/band.py --rho 0.25,0.5,1,2 --out $O/sweep_spin.json > $O/sweep_spin.log 2>&1; echo sweep rc=$?
timeout 900 $R --master-port 29506 tools/band.py --rho 0.25,0.5,1,2 --compute gemm --out $O/sweep_gemm.json > $O/sweep_gemm.log 2>&1; echo sweep_gemm rc=$?
