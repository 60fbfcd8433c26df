python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out/n2c; mkdir -p $O
for m in bucket p2p ce; do
  timeout 300 $R --master-port 29641 bench.py --gpus 2 --config mlp --steps 200 --warmup 10 --sync-mode $m > $O/mlp_graph_$m.json 2> $O/mlp_graph_$m.err; echo mlp $m rc=$?
done
timeout 600 $R --master-port 29642 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 600 $R --master-port 29643 tools/band.py --rho 0.1,0.15,0.2 --scenario-band --out $O/band_spin.json > $O/band_spin.log 2>&1; echo band rc=$?
