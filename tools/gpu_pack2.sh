python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out/pack; mkdir -p $O
for cap in 148 64; do
timeout 600 $R --master-port 29663 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-ctas $cap --out $O/band_gemm_cap$cap.json > $O/band_gemm_cap$cap.log 2>&1; echo cap$cap rc=$?
timeout 600 $R --master-port 29664 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-ctas $cap --pack-engine ce --out $O/band_gemm_cap${cap}_ce.json > $O/band_gemm_cap${cap}_ce.log 2>&1; echo cap${cap}ce rc=$?
done
