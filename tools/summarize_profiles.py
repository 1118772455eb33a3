"""Dev tool: turns the ncu artefacts brought back in gpurun_out/ into the tracked files under profiles/.

    python tools/summarize_profiles.py r01a C3 gpurun_out/launches_c3.csv gpurun_out/prof_factor.ncu-rep [gpurun_out/prof_tri.ncu-rep]
"""
import collections, csv, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
WANT = ["gpu__time_duration.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "smsp__cycles_active.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            us = v / 1e3 if d["Metric Unit"] in ("ns", "nsecond") else v
            a = agg.setdefault(d["Kernel Name"].split("(")[0], [0, 0.0])
            a[0] += 1
            a[1] += us
    return agg


def raw_metrics(rep, kernel_regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if kernel_regex not in d.get("Kernel Name", "") or "arm_" in d.get("Kernel Name", ""):
            continue
        res.append({w: (d[w], units[hdr.index(w)]) for w in WANT if w in d} | {"kernel": d["Kernel Name"]})
    return res


def source_top(rep, kernel_regex, n=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kernel_regex],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, body = None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if hdr is not None:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and r:
            body.append(r)
    idx = {k: i for i, k in enumerate(hdr)}
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(int(r[idx["# Samples"]]) for r in body) or 1
    agg = {k: sum(int(r[idx[k]]) for r in body) for k in stalls}
    top = sorted(body, key=lambda r: -int(r[idx["# Samples"]]))[:n]
    lines = [f"{int(r[idx['# Samples']]) / tot:6.3f}  {r[idx['Source']].strip()[:80]}" for r in top]
    return tot, sorted(agg.items(), key=lambda kv: -kv[1])[:6], lines


def main():
    tag, workload, launch_csv, *reps = sys.argv[1:]
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(launch_csv, os.path.join(PROF, f"{tag}_launches_{workload}.csv"))
    agg = launches(launch_csv)
    tot = sum(a[1] for a in agg.values())
    md = [f"# {tag}: ncu summary, workload {workload}", "",
          "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400` over "
          f"`bench.py --steps 2 --warmup 3` (cold-cache, serialised: compare SHARES). Raw: `{tag}_launches_{workload}.csv`.", "",
          "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k.strip()[:70]}` | {c} | {t:.1f} | {t / tot:.3f} | {t / c:.1f} |")
    traffic = {}
    seen = set()
    for rep in reps:
        for kr in ("factor_kernel", "factor_block_kernel", "factor_block_team_kernel", "factor_tile_kernel", "tri_kernel", "tri_upper_team_kernel", "tail_kernel"):
            ms = raw_metrics(rep, kr)
            if not ms:
                continue
            md += ["", f"## `{kr}` — `ncu --set full --clock-control none --import-source on` ({os.path.basename(rep)})", ""]
            for m in ms[:2]:
                md.append(f"* `{m['kernel'][:90]}`")
                for w in WANT:
                    if w in m:
                        md.append(f"  * {w} = {m[w][0]} {m[w][1]}")
                if kr in ("factor_kernel", "factor_block_kernel", "factor_block_team_kernel", "factor_tile_kernel") and "dram__bytes_read.sum" in m and kr not in seen:
                    # one refactorization = the head launch + the row-blocked trailing launch: their traffic adds up
                    seen.add(kr)
                    def mb(x):
                        v, u = x
                        v = float(v.replace(",", ""))
                        return v * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[u]
                    traffic["factor_kernel_dram_bytes"] = traffic.get("factor_kernel_dram_bytes", 0.0) + \
                        mb(m["dram__bytes_read.sum"]) + mb(m["dram__bytes_write.sum"])
            try:
                tot_s, stalls, lines = source_top(rep, kr)
                md += ["", f"Stall samples ({tot_s} total): " + ", ".join(f"{k}={v}" for k, v in stalls), "",
                       "Top instructions by samples (share, SASS):", "", "```"] + lines + ["```"]
            except Exception as e:  # noqa
                md.append(f"(source page unavailable: {e})")
    open(os.path.join(PROF, f"{tag}_summary_{workload}.md"), "w").write("\n".join(md) + "\n")
    tp = os.path.join(PROF, "traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    if traffic:
        cur[workload] = traffic | {"source": f"profiles/{tag}_summary_{workload}.md"}
        json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(md[:30]))


if __name__ == "__main__":
    main()
