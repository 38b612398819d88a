"""Summarise the ncu captures of scripts/ncu_profile.sh into committed evidence under profiles/:

  profiles/<round>/ncu_<kernel>.json   key counters of each --set full capture
  profiles/<round>/launch_shares.md    per-kernel share of one bench step (launch list)
  profiles/ncu_traffic.json            DRAM bytes per forward-GEMM launch (read by bench.py)

Usage: python scripts/summarize_profiles.py gpurun_out profiles/r01 [launches_per_step]
"""
import collections
import csv
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
    "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = f"{vals[i]} {units[i]}".strip()
    return d


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    for rep in sorted(os.listdir(src)):
        if rep.startswith("prof_") and rep.endswith(".ncu-rep") and rep in (
                "prof_fwd_gate.ncu-rep", "prof_bwd_gate.ncu-rep", "prof_tok.ncu-rep", "prof_u.ncu-rep",
                "prof_preshrink.ncu-rep", "prof_dec3_q.ncu-rep", "prof_dec3_qkv.ncu-rep"):
            d = raw(os.path.join(src, rep))
            with open(os.path.join(dst, "ncu_" + rep[5:-8] + ".json"), "w") as f:
                json.dump(d, f, indent=1)
    # the library's launches (kernels in namespace smlm, incl. the plan-copy kernel); the timed
    # step is the last `per_step` of them (bench.py --steps 1 --warmup 1; gpu_launches / steps)
    per_step = int(sys.argv[3]) if len(sys.argv) > 3 else 69
    data = [d for d in launches(os.path.join(src, "launches.csv")) if "smlm" in d["Kernel Name"]]
    step = data[-per_step:]
    agg = collections.OrderedDict()
    for d in step:
        k = d["Kernel Name"].split("(")[0].replace("void smlm::<unnamed>::", "").replace("smlm::<unnamed>::", "")
        agg[k] = agg.get(k, 0.0) + float(d["Metric Value"]) / 1000.0
    tot = sum(agg.values())
    with open(os.path.join(dst, "launch_shares.md"), "w") as f:
        f.write("# Kernel shares of one C4 layer-step (ncu launch list, serialised, cold cache)\n\n")
        f.write(f"{len(step)} launches, {tot:.1f} us summed device time\n\n| us | share | kernel |\n|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1]):
            f.write(f"| {v:.1f} | {100 * v / tot:.1f}% | `{k}` |\n")
    tr = launches(os.path.join(src, "fwd_traffic.csv"))
    per = collections.defaultdict(dict)
    for d in tr:
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"])
    byts = [v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values()]
    if byts:
        with open(os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json"), "w") as f:
            json.dump({"fwd_gemm_dram_bytes_per_launch": sum(byts) / len(byts),
                       "per_launch_bytes": byts, "launches": len(byts),
                       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the 7 forward "
                                 "smlm_gemm2_kernel launches of one bench step (scripts/ncu_profile.sh)"}, f, indent=1)
    print(open(os.path.join(dst, "launch_shares.md")).read())


if __name__ == "__main__":
    main()
