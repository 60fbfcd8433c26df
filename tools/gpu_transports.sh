# Which transport beside tensor-core compute: the GEMM band at N = 4 with the same buckets for
# every transport (absolute crossover rotation times).  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/transports; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for m in ce p2p p2p_gather nvls; do
  i=$((i+1))
  X=""; [ $m = nvls ] && X="--sync-ctas 148"
  timeout 600 $R --master-port 2995$i tools/band.py --sizes-mb 350,700,1400 --compute gemm --sync-mode $m --steps 60 --energy $X --out $O/band_gemm_${m}_n4.json > $O/band_gemm_${m}_n4.log 2>&1; echo band $m rc=$?
done
