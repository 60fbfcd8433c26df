# Round-2 power accounting (profiles/r02_power): the GEMM band and the spin band at N = 4 with the
# board energy counter around every timed region.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/power2; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29921 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-mode nvls --sync-ctas 148 --steps 100 --energy --out $O/band_gemm_nvls_n4.json > $O/band_gemm_nvls_n4.log 2>&1; echo gemm nvls rc=$?
timeout 600 $R --master-port 29922 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-mode ce --steps 100 --energy --out $O/band_gemm_ce_n4.json > $O/band_gemm_ce_n4.log 2>&1; echo gemm ce rc=$?
timeout 600 $R --master-port 29923 tools/band.py --rho 0.5,1 --sync-mode nvls --steps 100 --energy --out $O/band_spin_nvls_n4.json > $O/band_spin_nvls_n4.log 2>&1; echo spin nvls rc=$?
