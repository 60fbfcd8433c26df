# GEMM band at N = 4, p2p transport, the same bucket sizes: capped kernel on the TMA ring vs in
# registers (A/B of the sync's effect on a TMA-fed GEMM).  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/bandbulk2; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in bulk registers; do
  X=""; [ $v = registers ] && X="--p2p-registers"
  timeout 600 $R --master-port 2987$([ $v = bulk ] && echo 2 || echo 3) tools/band.py --sizes-mb 350,700,1400 --compute gemm --sync-mode p2p --steps 60 --energy $X --out $O/band_gemm_p2p_${v}_n4.json > $O/band_gemm_p2p_${v}_n4.log 2>&1; echo band $v rc=$?
  timeout 600 $R --master-port 2988$([ $v = bulk ] && echo 2 || echo 3) tools/band.py --sizes-mb 350,700,1400 --compute spin --sync-mode p2p --steps 60 $X --out $O/band_spin_p2p_${v}_n4.json > $O/band_spin_p2p_${v}_n4.log 2>&1; echo spin $v rc=$?
done
