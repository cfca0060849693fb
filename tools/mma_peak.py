"""Tensor-pipe ceiling of this B200 (``tnx_mma_peak``): MMA-only loops of
tcgen05.mma kind::tf32 and kind::f16 (BF16), cta_group 1 and 2, burst
(~50 ms) and sustained (~5 s), with the SM clock the CTAs measured.

    python tools/mma_peak.py [--sustained-s 5] [--out profiles/r02_mma_peak.json]

The GEMM roofline divides by the TF32 figure / 3 (split-TF32: 3 real MMA
passes per complex product term; 8 M N K complex flop = 24 M N K real
tensor-core flop).  Also prints flop/clk/SM so the ceiling can be rescaled to
any sampled clock.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2002_01935_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sustained-s", type=float, default=5.0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []
    for kind in ("tf32", "bf16"):
        for cg in (1, 2):
            # calibrate: iterations for ~50 ms
            t, mhz, ms = _native.mma_peak(kind, cg, 20000)
            it = max(1000, int(20000 * 50.0 / max(ms, 1e-3)))
            t, mhz, ms = _native.mma_peak(kind, cg, it)
            rows.append({"kind": kind, "cta_group": cg, "mode": "burst", "iters": it, "ms": ms,
                         "tflops": t, "sm_mhz": mhz, "flop_per_clk_per_sm": t * 1e12 / (mhz * 1e6) / sms})
            print(json.dumps(rows[-1]), flush=True)
    t, mhz, ms = _native.mma_peak("ffma", 1, 20000)
    it = max(1000, int(20000 * 50.0 / max(ms, 1e-3)))
    t, mhz, ms = _native.mma_peak("ffma", 1, it)
    rows.append({"kind": "ffma", "cta_group": 0, "mode": "burst", "iters": it, "ms": ms, "tflops": t,
                 "sm_mhz": mhz, "flop_per_clk_per_sm": t * 1e12 / (mhz * 1e6) / sms})
    print(json.dumps(rows[-1]), flush=True)
    if args.sustained_s > 0:
        for kind in ("tf32",):
            for cg in (2,):
                t, mhz, ms = _native.mma_peak(kind, cg, 20000)
                it = int(20000 * args.sustained_s * 1e3 / ms)
                t, mhz, ms = _native.mma_peak(kind, cg, it)
                rows.append({"kind": kind, "cta_group": cg, "mode": "sustained", "iters": it, "ms": ms,
                             "tflops": t, "sm_mhz": mhz, "flop_per_clk_per_sm": t * 1e12 / (mhz * 1e6) / sms})
                print(json.dumps(rows[-1]), flush=True)
    best = max((r for r in rows if r["kind"] == "tf32" and r["mode"] == "burst"), key=lambda r: r["tflops"])
    summary = {"device": torch.cuda.get_device_name(0), "sms": sms, "rows": rows,
               "tf32_peak_tflops": best["tflops"], "tf32_peak_sm_mhz": best["sm_mhz"],
               "complex_3xtf32_peak_tflops": best["tflops"] / 3.0,
               "ffma_tflops": rows[4]["tflops"] if len(rows) > 4 else None}
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
