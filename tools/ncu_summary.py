"""Summarise an ncu report (k_match) and a launch list into profiles/: python tools/ncu_summary.py <tag> <workload>"""
import csv, io, json, os, subprocess, sys, collections

tag, workload = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = os.path.join(root, "gpurun_out", f"prof_{tag}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__sectors_read.sum",
        "dram__sectors_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct", "lts__t_sectors_data_ecc.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size"]
m = {}
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            m[w] = (vals[i], units[i])
with open(os.path.join(root, "profiles", f"{tag}_k_match_full_raw.csv"), "w") as f:
    f.write(raw)
def num(k):
    v, u = m[k]
    x = float(v.replace(",", ""))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(u, 1)
    return x * scale
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
# the bench line of the profiled run names the exact configuration: traffic.json is keyed like
# bench.py's traffic_key (workload/layout/k/reads per GPU) and holds DRAM bytes per read
line = json.loads([ln for ln in open(os.path.join(root, "gpurun_out", f"prof_{tag}.json")).read().splitlines() if ln.startswith("{")][-1])
cfgj = line["config"]
Q = cfgj["reads_per_gpu"]
key = f"{workload}/{line['layout']}/k{cfgj['kmer_k']}/Q{Q}"
tr_path = os.path.join(root, "profiles", "traffic.json")
tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
tr = {k: v for k, v in tr.items() if isinstance(v, dict)}  # (drop the r01 flat entries)
tr[key] = {"dram_bytes_per_read": dram / Q, "dram_bytes_per_launch": dram,
           "source": f"profiles/{tag}_k_match_full_raw.csv (ncu --set full, one k_match launch of bench.py)"}
json.dump(tr, open(tr_path, "w"), indent=1)
# launch list shares
txt = open(os.path.join(root, "gpurun_out", f"launches_{tag}.csv")).read()
txt = txt[txt.index('"ID"'):]
agg = collections.OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")[:80]
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += float(r["Metric Value"])
lines = [f"# {tag}: ncu summary ({workload})", "", "| metric | value |", "|---|---|"]
lines += [f"| {k} | {v} {u} |" for k, (v, u) in m.items()]
lines += ["", f"dram read+write per launch: {dram/1e9:.2f} GB = {dram/Q:.1f} B per read ({key})", "", "Launch list (ncu gpu__time_duration.sum, serialised):", "",
          "| kernel | launches | total ms |", "|---|---|---|"]
lines += [f"| {k} | {c} | {t/1e6:.3f} |" for k, (c, t) in agg.items()]
# the bench steps only (from the first read-ordering launch on): each kernel's share of a step
rows = list(csv.DictReader(io.StringIO(txt)))
first = next((i for i, r in enumerate(rows) if "k_presort_keys" in r["Kernel Name"]), None)
if first is not None:
    step = collections.OrderedDict()
    import re
    for r in rows[first:]:
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")[:80]
        if re.search(r"k_match\w*<[^>]*?, 1[,>]", name) and re.search(r"k_match<\d+, \d+, 1", name):
            break  # the instrumented (SA_MATCH_STATS) launch after the timed steps
        if not any(x in name for x in ("k_presort_keys", "DeviceRadixSort", "k_match")):
            continue
        a = step.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += float(r["Metric Value"])
    tot = sum(t for _, t in step.values())
    lines += ["", "Timed steps only (ordering + match launches of bench.py's steps; ncu, serialised, cold caches):", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    lines += [f"| {k} | {c} | {t/1e6:.3f} | {t/tot:.3f} |" for k, (c, t) in step.items()]
open(os.path.join(root, "profiles", f"{tag}_SUMMARY.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
