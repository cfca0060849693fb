"""Same GEMM (M=N=8192, K=4096, 3xTF32) with random vs low-entropy operands,
run back to back for ~2 s each: per-launch time and (separately sampled)
clocks / power show whether the data-dependent power draw caps the clock."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
kind = sys.argv[1] if len(sys.argv) > 1 else "random"
rng = np.random.default_rng(0)
ml = [f"m{i}" for i in range(13)]; nl = [f"n{i}" for i in range(13)]; kl = [f"k{i}" for i in range(12)]
tab = {l: 2 for l in ml + nl + kl + ["s"]}
shx, shy = (2,) * 26, (2,) * 26
if kind == "random":
    x = rng.standard_normal(shx) + 1j * rng.standard_normal(shx)
    y = rng.standard_normal(shy) + 1j * rng.standard_normal(shy)
else:  # circuit-like: entries from {0, +-1/sqrt2, +-i/sqrt2}
    vals = np.array([0, 1, -1, 1j, -1j]) / np.sqrt(2)
    x = vals[rng.integers(0, 5, shx)]
    y = vals[rng.integers(0, 5, shy)]
tn = TensorNetwork([TensorNode(0, ml + kl, x), TensorNode(1, nl + kl, y)], tab, tuple(ml + nl))
plan = SlicedPlan(tn, ContractionTree((0, 1), [(0, 1)]), ()).bind()
import subprocess
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "50"], stdout=subprocess.PIPE, text=True)
ts = []
t0 = time.time()
while time.time() - t0 < 6.0:
    ts += [t for k, v, t in plan.profile_slice(0) if k == "gemm"]
smi.terminate()
samples = [tuple(float(x) for x in ln.split(",")) for ln in smi.stdout.read().splitlines() if ln.strip()]
clk = np.array([c for c, p in samples[len(samples) // 5:]])
pw = np.array([p for c, p in samples[len(samples) // 5:]])
print(f"{kind}: SM clock median {np.median(clk):.0f} MHz (min {clk.min():.0f}), power median {np.median(pw):.0f} W "
      f"(max {pw.max():.0f})")
ts = np.array(ts)
print(f"{kind}: {len(ts)} launches, median {np.median(ts):.3f} ms = {8 * 2**38 / np.median(ts) / 1e9:.1f} TF/s, "
      f"min {ts.min():.3f} ms")
