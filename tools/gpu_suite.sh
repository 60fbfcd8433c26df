# full -m gpu suite + smoke + the 8-rank peer-transport parity on one GPU
python -c "import sys; sys.path.insert(0,'.'); from paper_2103_07974_b200 import _build; _build.build(force=True)" || exit 1
O=gpurun_out/suite; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -2 $O/smoke.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29780 tests/mp_peer_check.py $O/peer_w8.json parity > $O/peer_w8.log 2>&1; echo peer_w8 rc=$?
python -c "import json,sys; d=json.load(open(\"$O/peer_w8.json\")); print(\"peer_w8 ok\", d[\"ok\"])"
