"""Turn a gpu_round.sh session (gpurun_out/) into the tracked summaries under
profiles/: the per-kernel launch-list shares, the GEMM and permute ncu
full-capture summaries (time, DRAM traffic vs algorithmic bytes, pipe
utilisation) and copies of the bench JSON lines.

    python tools/summarize_profiles.py [gpurun_out] [profiles] [round tag, e.g. r01]
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles"
TAG = sys.argv[3] if len(sys.argv) > 3 else "r01"


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return [dict(zip(head, r)) for r in rows[2:]], dict(zip(head, units))


def scaled(d, units, key):
    """Metric value in base units (bytes, seconds, Hz)."""
    v = float(d[key])
    u = units.get(key, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
            "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}
    return v * mult.get(u, 1)


def get(d, *keys):
    for k in keys:
        if k in d and d[k] not in ("", "n/a"):
            return d[k]
    return None


def launches():
    path = os.path.join(SRC, "launches.csv")
    if not os.path.exists(path):
        return
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        if "Kernel Name" not in r:
            continue
        name = (r["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
                .split("(")[0].split("<")[0].replace("void ", "").replace("tnx::", ""))
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        tot[name] += v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        cnt[name] += 1
    s = sum(tot.values())
    summ = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 "
                       "--warmup 3 --no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0",
            "note": "cold-cache serialised per-launch times (bind+hoist, warmup+timed slices, profile_slice); "
                    "compare shares, not absolutes",
            "kernels": [{"kernel": k, "launches": cnt[k], "total_ms": round(tot[k], 3),
                         "share": round(tot[k] / s, 4)} for k in sorted(tot, key=lambda k: -tot[k])]}
    shutil.copy(path, os.path.join(DST, f"{TAG}_launches.csv"))
    json.dump(summ, open(os.path.join(DST, f"{TAG}_launches_summary.json"), "w"), indent=1)
    print("launches:", [(k["kernel"], k["share"]) for k in summ["kernels"][:4]])


def gemm():
    rep = os.path.join(SRC, "prof_gemm_full.ncu-rep")
    if not os.path.exists(rep):
        return
    rows, units = raw_rows(rep)
    d = rows[0]
    t = scaled(d, units, "gpu__time_duration.sum")
    rd = scaled(d, units, "dram__bytes_read.sum")
    wr = scaled(d, units, "dram__bytes_write.sum")
    M, N, K = (int(x) for x in os.environ.get("GEMM_SHAPE", "8192 8192 4096").split())
    # operand planes read once + c64 output: A 4 fp32 planes; B 4, or 6 for the
    # stacked-B instance (template argument 4 = 1: -im_hi, -im_lo planes)
    name = d["Kernel Name"]
    i0 = name.find("kernel<")
    targs = name[i0 + 7:name.find(">", i0)].split(",") if i0 >= 0 else []
    stacked = len(targs) >= 4 and targs[3].strip() in ("1", "true")
    alg = 16 * M * K + (24 if stacked else 16) * K * N + 8 * M * N
    flops = 8 * M * N * K
    out = {"kernel": d["Kernel Name"],
           "command": "ncu --set full --clock-control none --import-source on -k regex:gemm_c64 -c 1 "
                      f"python tools/run_gemm.py {M} {N} {K} 1 1",
           "shape": [M, N, K],
           "sm_clock_ghz": scaled(d, units, "sm__cycles_elapsed.avg.per_second") / 1e9,
           "duration_ms": t * 1e3,
           "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "algorithmic_bytes": alg, "traffic_over_algorithmic": (rd + wr) / alg,
           "flops_8MNK": flops, "achieved_tflops_complex_at_ncu_clock": flops / t / 1e12,
           "tensor_pipe_active_pct": float(get(d, "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active",
                                              "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                                              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") or "nan"),
           "lts_throughput_pct": float(get(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed") or "nan"),
           "dram_throughput_pct": float(get(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                                            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or "nan"),
           "registers_per_thread": int(float(d["launch__registers_per_thread"])),
           "grid": d.get("launch__grid_size"), "cluster": "x".join(
               d.get(f"launch__cluster_dim_{a}", "1") for a in "xyz")}
    json.dump(out, open(os.path.join(DST, "ncu_gemm_traffic.json"), "w"), indent=1)
    shutil.copy(rep, os.path.join(DST, f"{TAG}_gemm_full.ncu-rep"))
    print("gemm:", round(out["duration_ms"], 3), "ms", round(out["achieved_tflops_complex_at_ncu_clock"], 1), "TF/s")


def perm():
    rep = os.path.join(SRC, "prof_perm_full.ncu-rep")
    if not os.path.exists(rep):
        return
    rows, units = raw_rows(rep)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else None
    ks = []
    for d in rows:
        t = scaled(d, units, "gpu__time_duration.sum")
        rd = scaled(d, units, "dram__bytes_read.sum")
        wr = scaled(d, units, "dram__bytes_write.sum")
        name = d["Kernel Name"].split("(")[0]
        # tools/run_perm.py: one slice of x = 4^13 complex64 elements
        n = 4 ** 13
        alg = 8 * n * 2 if name.startswith("gather") else 8 * n + 16 * n
        ks.append({"kernel": name, "duration_us": t * 1e6, "dram_read": rd, "dram_write": wr,
                   "algorithmic_bytes": alg, "achieved_gbs_algorithmic": alg / t / 1e9,
                   "dram_gbs": (rd + wr) / t / 1e9,
                   "frac_of_measured_hbm": (alg / t / 1e9) / peak if peak else None,
                   "dram_active_pct": float(d.get("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "nan")),
                   "registers_per_thread": int(float(d["launch__registers_per_thread"])),
                   "achieved_occupancy_pct": float(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "nan")),
                   "smem_bank_conflicts": d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")})
    out = {"workload": "tools/run_perm.py: x[s, m0,k0,...,m5,k5,m6] (13 dim-4 labels + sliced dim-2 label) "
                       "packed into K-blocked split-TF32 GEMM planes every slice: 2^26 complex64 in, "
                       "4 x 2^26 fp32 out; the gather copies the slice of the sliced leaf",
           "command": "ncu --set full --clock-control none --import-source on -k regex:'perm|gather' -c 2 "
                      "python tools/run_perm.py 1",
           "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)",
           "kernels": ks}
    json.dump(out, open(os.path.join(DST, "ncu_perm_traffic.json"), "w"), indent=1)
    shutil.copy(rep, os.path.join(DST, f"{TAG}_perm_full.ncu-rep"))
    print("perm:", [(k["kernel"], round(k["duration_us"], 1), round(k["achieved_gbs_algorithmic"])) for k in ks])


def simt():
    rep = os.path.join(SRC, "prof_simt_full.ncu-rep")
    if not os.path.exists(rep):
        return
    rows, units = raw_rows(rep)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else None
    # tools/run_simt.py: (a) x 2^24 + y 2^4 read, 2^20 written; (b) x 2^24 + y 2^14 read, 2^10 written (complex64)
    algs = [8 * (2 ** 24 + 2 ** 4 + 2 ** 20), 8 * (2 ** 24 + 2 ** 14 + 2 ** 10)]
    ks = []
    for d, alg, case in zip(rows, algs, ["skinny: 2^20 outputs x 16 terms (batched SIMT, thread mode)",
                                         "long sums: 2^10 outputs x 2^14 terms (split mode)"]):
        t = scaled(d, units, "gpu__time_duration.sum")
        rd = scaled(d, units, "dram__bytes_read.sum")
        wr = scaled(d, units, "dram__bytes_write.sum")
        ks.append({"case": case, "kernel": d["Kernel Name"].split("(")[0], "duration_us": t * 1e6,
                   "dram_read": rd, "dram_write": wr, "algorithmic_bytes": alg,
                   "achieved_gbs_algorithmic": alg / t / 1e9,
                   "frac_of_measured_hbm": (alg / t / 1e9) / peak if peak else None,
                   "registers_per_thread": int(float(d["launch__registers_per_thread"]))})
    out = {"command": "ncu --set full --clock-control none --import-source on -k regex:simt -c 2 "
                      "python tools/run_simt.py 1", "peak_gbs": peak, "kernels": ks}
    json.dump(out, open(os.path.join(DST, "ncu_simt_traffic.json"), "w"), indent=1)
    shutil.copy(rep, os.path.join(DST, f"{TAG}_simt_full.ncu-rep"))
    print("simt:", [(k["kernel"], round(k["duration_us"], 1), round(k["achieved_gbs_algorithmic"])) for k in ks])


def inslice_traffic():
    """DRAM bytes of every tensor-core launch of one bench slice (ncu launch
    list with dram metrics + the bench's --profile-out vertex list) against the
    kernel's algorithmic bytes: operand planes read once (16 B per A element,
    24 B per stacked-B / 16 B per B element) + the result written once (8 B
    complex64, 16 B direct planes)."""
    path = os.path.join(SRC, "launches_dram.csv")
    prof_path = os.path.join(SRC, "profile.json")
    if not (os.path.exists(path) and os.path.exists(prof_path)):
        return
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = defaultdict(dict), {}
    for r in rows[hi + 1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki]
    prof = json.load(open(prof_path))
    verts = {v["ssa"]: v for v in prof["vertices"]}
    gl = [l for l in prof["launches"] if l[0] == "gemm"]
    g_ids = [i for i in sorted(per) if "gemm_c64" in names[i]][-len(gl):]
    out = []
    for l, i in zip(gl, g_ids):
        x = verts[l[1]]
        b, m, n, k = x["batch"], x["m"], x["n"], x["k"]
        kp = (k + 15) // 16 * 16
        ta = names[i].split("kernel<")[1].split(">")[0].split(",")
        epi, stacked = ta[2].strip(), ta[3].strip() == "1"
        alg = 16 * b * m * kp + (24 if stacked else 16) * b * n * kp + (8 if epi == "0" else 16) * b * m * n
        dram = per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"]
        out.append({"ssa": l[1], "M": m, "N": n, "K": k, "batch": b, "epilogue": int(epi), "stacked_b": stacked,
                    "ms_ncu": per[i]["gpu__time_duration.sum"] / 1e6, "dram_bytes": dram, "algorithmic_bytes": alg,
                    "ratio": dram / alg})
    out.sort(key=lambda r: -r["ms_ncu"])
    td, ta_ = sum(r["dram_bytes"] for r in out), sum(r["algorithmic_bytes"] for r in out)
    summ = {"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                       "sm__cycles_elapsed.max --clock-control none python bench.py --steps 1 --warmup 0 "
                       "--no-cpu-baseline --no-e2e --no-tf32-probe --sustained-s 0 --profile-out profile.json",
            "note": "last profiled slice's tensor-core launches (cold-cache, serialised by ncu)",
            "dominant": out[0], "all_gemm_dram_bytes": td, "all_gemm_algorithmic_bytes": ta_,
            "all_gemm_ratio": td / ta_, "launches": out}
    json.dump(summ, open(os.path.join(DST, f"{TAG}_gemm_inslice_traffic.json"), "w"), indent=1)
    print("in-slice gemm traffic: dominant ratio", round(out[0]["ratio"], 2), "all", round(td / ta_, 2))


def benches():
    for src, dst in [("bench_default.log", f"{TAG}_bench_default.json"),
                     ("bench_sustained.log", f"{TAG}_bench_long.json"),
                     ("bench_reference.log", f"{TAG}_bench_reference.json"),
                     ("bench_2rank_gloo.log", f"{TAG}_bench_2rank_gloo_shared_gpu.json")]:
        p = os.path.join(SRC, src)
        if os.path.exists(p):
            line = [ln for ln in open(p) if ln.startswith("{")][-1]
            json.dump(json.loads(line), open(os.path.join(DST, dst), "w"), indent=1)


if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    launches()
    inslice_traffic()
    gemm()
    perm()
    simt()
    benches()
