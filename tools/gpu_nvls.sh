python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/nvb; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29921 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --sync-mode nvls > $O/bench_nvls.json 2> $O/bench_nvls.err; echo bench rc=$?
timeout 600 $R --master-port 29922 tools/band.py --rho 0.5,1,2 --sync-mode nvls --out $O/sweep_spin_nvls.json > $O/sweep_spin_nvls.log 2>&1; echo spin rc=$?
timeout 600 $R --master-port 29923 tools/band.py --rho 0.2,0.5,1 --compute gemm --sync-ctas 148 --sync-mode nvls --out $O/band_gemm_nvls.json > $O/band_gemm_nvls.log 2>&1; echo gemm rc=$?
timeout 600 $R --master-port 29924 bench.py --gpus 4 --steps 20 --warmup 5 --mix resnet50:8,vgg16:2 --sync-mode nvls > $O/mix_nvls.json 2> $O/mix_nvls.err; echo mix rc=$?
