"""Diagnose run-to-run variation of the ResNet-50 + VGG-16 + BERT crossover mix.

    torchrun --nproc-per-node 4 tools/diag_mix3.py
"""
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import Harness, timed_run  # noqa: E402


def main():
    from paper_2103_07974_b200 import apps
    from paper_2103_07974_b200.engine import Phase
    from paper_2103_07974_b200.scheduler import Policy

    h = Harness()
    dev, rank = h.dev, h.rank
    base = [apps.resnet50_app("r", 256, 1, dev, seed=rank, graphed=True, flat="ipc", fast_bn=True),
            apps.vgg16_app("v", 64, 1, dev, seed=1000 + rank, graphed=True, flat="ipc", fast_bn=True),
            apps.bert_app("b", 32, 128, 1, dev, seed=2000 + rank, flat="ipc")]
    mode = sys.argv[1] if len(sys.argv) > 1 else "ce"
    for run in range(5):
        r = timed_run(h, base, Policy.CROSSOVER, 3, 10, sync_mode=mode, time_kernels=False)
        if rank == 0:
            per = {}
            for s in r["timed_spans"]:
                per.setdefault((s.job_id, s.phase), []).append((s.end - s.start) / 1e6)
            med = {f"{j}.{p.value[0]}": round(statistics.median(v), 2) for (j, p), v in sorted(per.items(), key=lambda kv: (kv[0][0], kv[0][1].value))}
            print(f"run {run}: {r['ms'] / 10:.2f} ms/rotation  {med}  mem {torch.cuda.memory_reserved() / 2**30:.1f} GiB", flush=True)
        del r
    h.close()


if __name__ == "__main__":
    main()
