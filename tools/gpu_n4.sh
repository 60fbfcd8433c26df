# 4-GPU round: NCCL multi-rank parity at W=2/4, bench N=4 (configs 2, 1, 3, 5), CE transport, band
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
O=gpurun_out/n4; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > $O/multirank.log 2>&1; echo multirank rc=$?
timeout 900 $R --master-port 29601 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 600 $R --master-port 29602 tools/cebench.py --sizes-mb 128,512 --out $O/cebench.json > $O/cebench.log 2>&1; echo cebench rc=$?
timeout 900 $R --master-port 29603 tools/band.py --rho 0.1,0.15,0.2 --scenario-band --out $O/band_spin.json > $O/band_spin.log 2>&1; echo band rc=$?
timeout 900 $R --master-port 29604 tools/band.py --rho 0.1,0.15,0.2,0.5,1 --compute gemm --scenario-band --out $O/band_gemm.json > $O/band_gemm.log 2>&1; echo band_gemm rc=$?
timeout 900 $R --master-port 29605 tools/band.py --rho 0.25,0.5,1,2 --out $O/sweep_spin.json > $O/sweep_spin.log 2>&1; echo sweep rc=$?
timeout 600 $R --master-port 29606 bench.py --gpus 4 --config mlp --steps 200 --warmup 10 > $O/bench_mlp.json 2> $O/bench_mlp.err; echo mlp rc=$?
for mix in resnet50:16,vgg16:4 resnet50:8,vgg16:2 resnet50:256,vgg16:64 resnet50:256,vgg16:64,bert:32; do
  timeout 900 $R --master-port 29607 bench.py --gpus 4 --steps 20 --warmup 5 --mix $mix > "$O/mix_$mix.json" 2> "$O/mix_$mix.err"; echo mix $mix rc=$?
done
