set -x
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b_n1.json 2> gpurun_out/b_n1.err; echo rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --sync-ctas -1 --no-cpu-baseline > gpurun_out/b_n1_cap.json 2> gpurun_out/b_n1_cap.err; echo rc=$?
timeout 600 python bench.py --config mlp --steps 200 --warmup 10 > gpurun_out/b_mlp_n1.json 2> gpurun_out/b_mlp_n1.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; echo rc=$?
timeout 600 python bench.py --impl reference --config mlp --steps 200 --warmup 10 > gpurun_out/ref_mlp_n1.json 2> gpurun_out/ref_mlp_n1.err; echo rc=$?
