python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out/pack; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -k copy_engines > $O/t.log 2>&1; echo test rc=$?; tail -1 $O/t.log
timeout 600 $R --master-port 29661 tools/band.py --rho 0.2,0.5,1 --compute gemm --pack-engine ce --out $O/band_gemm_ce.json > $O/band_gemm_ce.log 2>&1; echo ce rc=$?
timeout 600 $R --master-port 29662 tools/band.py --rho 0.2,0.5,1 --compute gemm --pack-engine sm --out $O/band_gemm_sm.json > $O/band_gemm_sm.log 2>&1; echo sm rc=$?
