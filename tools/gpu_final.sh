# Round-2 final measurement set (profiles/r02_final): configs 1 and 2 at N = 1 / 2 / 4, the
# speedup band, the reference arms.  Run under gpurun --gpus 4.
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/final; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo bench n1 rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_n1.json 2> $O/ref_n1.err; echo ref n1 rc=$?
timeout 600 python bench.py --config mlp --steps 300 --warmup 10 > $O/mlp_n1.json 2> $O/mlp_n1.err; echo mlp n1 rc=$?
timeout 600 python bench.py --impl reference --config mlp --steps 300 --warmup 10 > $O/ref_mlp_n1.json 2> $O/ref_mlp_n1.err; echo ref mlp rc=$?
for n in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 900 $R --master-port 2980$n bench.py --gpus $n --steps 20 --warmup 5 > $O/bench_n$n.json 2> $O/bench_n$n.err; echo bench n$n rc=$?
  timeout 600 $R --master-port 2981$n bench.py --gpus $n --config mlp --steps 300 --warmup 10 > $O/mlp_n$n.json 2> $O/mlp_n$n.err; echo mlp n$n rc=$?
  timeout 900 $R --master-port 2982$n tools/band.py --rho 0.1,0.15,0.2 --scenario-band --out $O/band_spin_n$n.json > $O/band_spin_n$n.log 2>&1; echo band n$n rc=$?
done
