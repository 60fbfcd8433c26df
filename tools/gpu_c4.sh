python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/c4; mkdir -p $O
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
timeout 900 $R --master-port 2969$n tools/band.py --sizes-mb 1,4,16,64,256,1024 --out $O/sizes_spin_n$n.json > $O/sizes_spin_n$n.log 2>&1; echo spin n$n rc=$?
timeout 900 $R --master-port 2969$n tools/band.py --sizes-mb 1,4,16,64,256,1024 --compute gemm --sync-ctas 148 --out $O/sizes_gemm_n$n.json > $O/sizes_gemm_n$n.log 2>&1; echo gemm n$n rc=$?
done
