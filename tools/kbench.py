"""Microbenchmark of K1/K2 variants at ResNet-50 / VGG-16 bucket sizes (device-timed).

    python tools/kbench.py [--model resnet50] [--iters 20]

Each timed launch is preceded by an L2 flush (write of a 512 MB buffer), so
every byte comes from HBM.  Reports algorithmic GB/s (SURVEY §8d bytes) and
the fraction of the measured HBM peak.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--only", default="", help="substring filter on case[variant] names")
    ap.add_argument("--sweep", action="store_true", help="sweep TMA launch shapes (cs_tune)")
    args = ap.parse_args()
    import torchvision

    from paper_2103_07974_b200 import _lib
    from paper_2103_07974_b200.fusion import FusedGradientSync, SgdSettings

    dev = torch.device("cuda", 0)
    m = getattr(torchvision.models, args.model)()
    shapes = [p.shape for p in m.parameters()]
    params = [torch.randn(s, device=dev) for s in shapes]
    grads = [torch.randn(s, device=dev) for s in shapes]
    S = sum(p.numel() for p in params) * 4
    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)
    clean = torch.ones(128 * 2**20, dtype=torch.float32, device=dev)

    def do_flush():
        # write 512 MB, then read 512 MB: L2 ends up holding clean lines only, so the
        # timed kernel pays neither cache hits nor somebody else's dirty write-backs
        flush.fill_(1)
        clean.sum()

    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    stream = torch.cuda.current_stream()

    def timeit(fn, iters):
        ts = []
        for _ in range(3):
            do_flush(); fn()
        for _ in range(iters):
            do_flush()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts), min(ts)

    res = {"model": args.model, "S_bytes": S, "peak_gbs": peak, "rows": []}
    src = torch.empty(S // 4, device=dev); dst = torch.empty_like(src)
    med, best = timeit(lambda: dst.copy_(src), args.iters)
    res["rows"].append({"name": "torch_copy(S)", "bytes": 2 * S, "us": med * 1e3, "GB/s": 2 * S / med / 1e6})
    cases = [
        ("k1_pack", dict(sgd=SgdSettings(0.1), mode="bucket", lw=1), "pack", 2 * S),
        ("k2_direct_momentum", dict(sgd=SgdSettings(0.1, momentum=0.9, weight_decay=1e-4), mode="direct", lw=1), "update", 5 * S),
        ("k2_bucket_momentum", dict(sgd=SgdSettings(0.1, momentum=0.9, weight_decay=1e-4), mode="bucket", lw=1), "update", 5 * S),
        ("k2_bucket_plain_ref", dict(sgd=SgdSettings(0.1), mode="bucket", lw=1), "update", 3 * S),
        ("k2_bucket_2src_momentum", dict(sgd=SgdSettings(0.1, momentum=0.9), mode="bucket", lw=2), "update", 6 * S),
    ]
    for variant_name, variant in (("tma", _lib.CS_VARIANT_TMA), ("register", _lib.CS_VARIANT_REGISTER)):
        _lib.set_kernel_variant(variant)
        for name, kw, what, nbytes in cases:
            if args.only and args.only not in f"{name}[{variant_name}]":
                continue
            s = FusedGradientSync(params, kw["sgd"], local_workers=kw["lw"], mode=kw["mode"])
            gl = [grads] * kw["lw"]
            if what == "pack":
                fn = lambda: s.pack(gl, stream.cuda_stream)
            elif kw["mode"] == "direct":
                fn = lambda: s.update(stream.cuda_stream, grads)
            else:
                s.pack(gl, stream.cuda_stream)
                fn = lambda: s.update(stream.cuda_stream)
            med, best = timeit(fn, args.iters)
            res["rows"].append({"name": f"{name}[{variant_name}]", "bytes": nbytes, "us": round(med * 1e3, 2),
                                "best_us": round(best * 1e3, 2), "GB/s": round(nbytes / med / 1e6, 1),
                                "frac_of_peak": round(nbytes / med / 1e6 / peak, 4)})
    if args.sweep:
        _lib.set_kernel_variant(_lib.CS_VARIANT_TMA)
        sm = FusedGradientSync(params, SgdSettings(0.1, momentum=0.9, weight_decay=1e-4), mode="direct")
        sp0 = FusedGradientSync(params, SgdSettings(0.1), mode="bucket")
        sp0.pack([grads], stream.cuda_stream)
        s2 = FusedGradientSync(params, SgdSettings(0.1, momentum=0.9), mode="bucket", local_workers=2)
        s2.pack([grads, grads], stream.cuda_stream)
        for cps in (1, 2):
            for chunk in (1024, 2048, 4096):
                for st in (0, 4):
                    _lib.tune("ctas_per_sm", cps); _lib.tune("k2_chunk", chunk); _lib.tune("k2_stages", st)
                    try:
                        med, best = timeit(lambda: sm.update(stream.cuda_stream, grads), args.iters)
                    except Exception as e:  # noqa: BLE001
                        print("sweep k2", cps, chunk, st, "failed", e); continue
                    res["rows"].append({"name": f"sweep_k2[cps={cps},chunk={chunk},stages={st or 'auto'}]",
                                        "bytes": 5 * S, "us": round(med * 1e3, 2), "GB/s": round(5 * S / med / 1e6, 1),
                                        "frac_of_peak": round(5 * S / med / 1e6 / peak, 4)})
        sp = FusedGradientSync(params, SgdSettings(0.1), mode="bucket")
        for cps in (1, 2):
            for chunk in (4096, 8192, 16384):
                _lib.tune("ctas_per_sm", cps); _lib.tune("k1_chunk", chunk)
                try:
                    med, best = timeit(lambda: sp.pack([grads], stream.cuda_stream), args.iters)
                except Exception as e:  # noqa: BLE001
                    print("sweep k1", cps, chunk, "failed", e); continue
                res["rows"].append({"name": f"sweep_k1[cps={cps},chunk={chunk}]", "bytes": 2 * S,
                                    "us": round(med * 1e3, 2), "GB/s": round(2 * S / med / 1e6, 1),
                                    "frac_of_peak": round(2 * S / med / 1e6 / peak, 4)})
        _lib.set_kernel_variant(_lib.CS_VARIANT_REGISTER)
        for shape in range(5):
            _lib.tune("reg_shape", shape)
            for nm, obj, fn2, nb in (("k2_direct_momentum", sm, lambda: sm.update(stream.cuda_stream, grads), 5 * S),
                                     ("k2_bucket_plain_ref", sp0, lambda: sp0.update(stream.cuda_stream), 3 * S),
                                     ("k2_bucket_2src_momentum", s2, lambda: s2.update(stream.cuda_stream), 6 * S),
                                     ("k1_pack", sp0, lambda: sp0.pack([grads], stream.cuda_stream), 2 * S)):
                med, best = timeit(fn2, args.iters)
                res["rows"].append({"name": f"reg_{nm}[shape={shape}]", "bytes": nb, "us": round(med * 1e3, 2),
                                    "GB/s": round(nb / med / 1e6, 1), "frac_of_peak": round(nb / med / 1e6 / peak, 4)})
        _lib.tune("reg_shape", 0)
        _lib.set_kernel_variant(_lib.CS_VARIANT_TMA)
        for dbg in (1, 2):
            for cps in (1, 2):
                _lib.tune("ctas_per_sm", cps); _lib.tune("k2_chunk", 2048); _lib.tune("k2_stages", 0)
                _lib.tune("k2_debug", dbg)
                med, best = timeit(lambda: sm.update(stream.cuda_stream, grads), args.iters)
                res["rows"].append({"name": f"ablate_k2[debug={dbg},cps={cps}]", "bytes": 5 * S,
                                    "us": round(med * 1e3, 2), "GB/s": round(5 * S / med / 1e6, 1)})
        _lib.tune("k2_debug", 0)
        for k in ("ctas_per_sm", "k2_chunk", "k2_stages", "k1_chunk"):
            _lib.tune(k, 0)
    for r in res["rows"]:
        print(f"{r['name']:40s} {r['us']:9.2f} us  {r['GB/s']:8.1f} GB/s  {r.get('frac_of_peak', '')}")
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
