"""Per-slot timeline of a 2-app synthetic crossover run (diagnosing transport choices).

    torchrun --nproc-per-node 4 tools/diag_adaptive.py <bucket MB> <sync mode>
"""
import sys, json
sys.path.insert(0, "/root/repo")
from bench import Harness, timed_run
from paper_2103_07974_b200.apps import synthetic_app
from paper_2103_07974_b200.scheduler import Policy
from paper_2103_07974_b200.engine import Phase
h = Harness()
mb = int(sys.argv[1]); mode = sys.argv[2]
base = [synthetic_app(f"syn{j}", mb * 2**20, 1, h.dev, gemm_reps=3, seed=j, flat="ipc") for j in range(2)]
r = timed_run(h, base, Policy.CROSSOVER, 3, 16, sync_mode=mode)
if h.rank == 0:
    sp = r["trace"].spans
    fw = [s for s in sp if s.phase is Phase.FORWARD]
    sy = [s for s in sp if s.phase is Phase.SYNC]
    print(mode, mb, "total ms", r["ms"], "tuner", r["sched"].tuner.summary() if r["sched"].tuner else None)
    print("fwd starts (ms):", [round((b.start - a.start) / 1e6, 2) for a, b in zip(fw, fw[1:])])
    print("sync dur (ms):", [round((s.end - s.start) / 1e6, 2) for s in sy])
    print("comp dur (ms):", [round((s.end - s.start) / 1e6, 2) for s in sp if s.phase is Phase.BACKWARD])
h.close()
