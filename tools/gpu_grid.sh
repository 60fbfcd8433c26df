python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out/grid; mkdir -p $O
timeout 600 $R --master-port 29631 tools/band.py --rho 0.1,0.2,0.5,1 --compute gemm --sync-ctas auto --out $O/band_gemm_auto.json > $O/band_gemm_auto.log 2>&1; echo band_auto rc=$?
timeout 600 $R --master-port 29632 tools/band.py --rho 0.1,0.2,0.5,1 --compute gemm --out $O/band_gemm_cap.json > $O/band_gemm_cap.log 2>&1; echo band_cap rc=$?
timeout 600 $R --master-port 29633 bench.py --gpus 2 --steps 20 --warmup 5 --mix resnet50:16,vgg16:4 --sync-ctas auto > $O/mix_auto.json 2> $O/mix_auto.err; echo mix rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --sync-ctas auto --no-cpu-baseline > $O/b_n1_auto.json 2> $O/b_n1_auto.err; echo n1 rc=$?
