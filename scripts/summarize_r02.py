"""Round-2 evidence under profiles/r02/ from the ncu captures of scripts/ncu_profile.sh
(gpurun_out/r02prof): key counters of each --set full capture, the per-kernel shares of one
C4 layer (launch list of scripts/prof_step.py), and the DRAM bytes of the CTA-pair GEMM launches
against their algorithmic bytes (-> profiles/ncu_traffic.json, read by bench.py)."""
import collections
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_profiles import KEYS, launches, raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r02prof")
dst = os.path.join(ROOT, "profiles", "r02")
os.makedirs(dst, exist_ok=True)
for rep in sorted(os.listdir(src)):
    if rep.startswith("prof_") and rep.endswith(".ncu-rep"):
        d = raw(os.path.join(src, rep))
        with open(os.path.join(dst, "ncu_" + rep[5:-8] + ".json"), "w") as f:
            json.dump(d, f, indent=1)


def us(d):
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    return v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)


# per-kernel shares of one layer (launch list)
data = launches(os.path.join(src, "launches_layer.csv"))
# the library's kernels only (not the workload set-up), of the second of the two steps
data = [d for d in data if "smlm::" in d["Kernel Name"]]
data = data[len(data) // 2:]
agg = collections.OrderedDict()
for d in data:
    k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("unnamed>::", "").replace("smlm::<", "")
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += us(d)
tot = sum(v[1] for v in agg.values())
lines = ["# One C4 layer (scripts/prof_step.py, layers=[0]): ncu launch list, per-kernel share",
         "", "ncu serialises launches and runs them cold: compare SHARES, not absolute times.", "",
         "| kernel | launches | us | share |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f} % |")
lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot:.1f} | |")
open(os.path.join(dst, "launch_shares.md"), "w").write("\n".join(lines) + "\n")

# CTA-pair GEMM DRAM traffic vs algorithmic bytes (C4: S rows, X/W/Y per launch group)
S, FT = 13448, 4096
alg = {   # forward: W + X + Y (+ unique B, small); backward: W + dY + dX (FT rows) + s*U
    "fwd q/k/v": 2 * (4096 * 6144 + S * 4096 + S * 6144),
    "fwd o": 2 * (4096 * 4096 + S * 4096 + S * 4096),
    "fwd gate/up": 2 * (4096 * 28672 + S * 4096 + S * 28672),
    "fwd down": 2 * (14336 * 4096 + S * 14336 + S * 4096),
    "bwd down": 2 * (14336 * 4096 + FT * 4096 + FT * 14336),
    "bwd gate/up": 2 * (28672 * 4096 + FT * 28672 + 2 * FT * 4096),
    "bwd o": 2 * (4096 * 4096 + FT * 4096 + FT * 4096),
    "bwd q/k/v": 2 * (6144 * 4096 + FT * 6144 + 3 * FT * 4096),
}
rows = list(csv.reader(open(os.path.join(src, "gemm_traffic.csv"))))
hdr, recs = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
out = []
for (name, ab), (i, m) in zip(alg.items(), recs.items()):
    b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    out.append({"launch": name, "dram_bytes": b, "alg_bytes": ab, "ratio": b / ab,
                "read": m["dram__bytes_read.sum"], "write": m["dram__bytes_write.sum"],
                "ncu_us": m["gpu__time_duration.sum"] / 1000.0})
fwd = [o for o in out if o["launch"].startswith("fwd")]
traffic = {"fwd_gemm_dram_bytes_per_launch": sum(o["dram_bytes"] for o in fwd) / len(fwd),
           "fwd_gemm_alg_bytes_per_launch": sum(o["alg_bytes"] for o in fwd) / len(fwd),
           "per_launch": out,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the 8 CTA-pair GEMM launches "
                     "of one C4 layer (scripts/prof_step.py; profiles/r02/gemm_traffic.csv)"}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
