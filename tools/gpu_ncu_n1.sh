# ncu evidence for the N=1 bench line: the launch list of the bench command and a full capture of K2
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:unpack_sgd -s 2 -c 2 -o gpurun_out/k2_n1 $CMD > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
