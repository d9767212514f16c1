"""Summarise the ncu outputs of scripts/gpu_bench_profile.sh into profiles/.

python scripts/ncu_summary.py TAG  ->  profiles/ncu_TAG_launches.csv (copy),
profiles/ncu_TAG_summary.md, profiles/ncu_traffic.json (dram bytes per launch)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
workload = sys.argv[2] if len(sys.argv) > 2 else "1B/M1/B1024"
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)
g = os.path.join(ROOT, "gpurun_out")

lines = []
lst = os.path.join(g, f"launches_{tag}.csv")
if os.path.exists(lst):
    shutil.copy(lst, os.path.join(out, f"ncu_{tag}_launches.csv"))
    txt = open(lst).read()
    body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(body)))
    per = {}
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            per.setdefault(name, []).append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in per.values())
    lines.append(f"## Launch list ({lst.split('/')[-1]}, ncu --metrics gpu__time_duration.sum --clock-control none)\n")
    lines.append("| kernel | launches | mean (us) | share of listed time |\n|---|---|---|---|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        unit = 1e-3 if max(v) > 1e4 else 1.0  # ns vs us
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) * unit:.1f} | {sum(v) / tot:.3f} |")
def emu_traffic(rep, traffic):
    """k_apply<M, ...> rows of the emulated-M capture -> traffic keys for M = 2, 4, 8."""
    import re

    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    hdr, units, data = rows[0], rows[1], rows[2:]
    ik, ir, iw, it = (hdr.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                              "gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for r in data:
        m = re.search(r"k_apply<(\d+)", r[ik])
        if not m:
            continue
        M = int(m.group(1))
        rd = float(r[ir].replace(",", "")) * scale.get(units[ir], 1)
        wr = float(r[iw].replace(",", "")) * scale.get(units[iw], 1)
        traffic[f"k_apply/{workload.split('/')[0]}/M{M}/B1024"] = {"dram_bytes_per_launch": rd + wr, "read": rd,
                                                                 "write": wr, "source": rep.split("/")[-1]}
        out.append((M, float(r[it].replace(",", "")), rd, wr))
    return out


traffic = {}
tpath = os.path.join(out, "ncu_traffic.json")
if os.path.exists(tpath):
    traffic = json.load(open(tpath))


def full_capture(rep, wl, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "smsp__inst_executed.sum", "lts__t_bytes.sum"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    lines.append(f"\n## ncu --set full ({rep.split('/')[-1]}{title})\n")
    lines.append("| metric | " + " | ".join(r[idx['Kernel Name']].split('(')[0].replace('void ', '') for r in data) + " |")
    lines.append("|---|" + "---|" * len(data))
    for w in want[1:]:
        if w in idx:
            lines.append(f"| {w} ({units[idx[w]]}) | " + " | ".join(r[idx[w]] for r in data) + " |")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        rd = float(r[idx["dram__bytes_read.sum"]].replace(",", "")) * scale.get(units[idx["dram__bytes_read.sum"]], 1)
        wr = float(r[idx["dram__bytes_write.sum"]].replace(",", "")) * scale.get(units[idx["dram__bytes_write.sum"]], 1)
        traffic[f"{name}/{wl}"] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                   "source": rep.split("/")[-1]}


rep = os.path.join(g, f"prof_{tag}.ncu-rep")
b0 = os.path.join(g, f"prof_b0_{tag}.ncu-rep")
if os.path.exists(b0):
    full_capture(b0, workload.replace("B1024", "B0"), ", B = 0: one scale per fragment, two passes")
if os.path.exists(rep):
    full_capture(rep, workload, "")
    emu = os.path.join(g, f"prof_emu_{tag}.ncu-rep")
    if os.path.exists(emu):
        rows = emu_traffic(emu, traffic)
        if rows:
            lines.append(f"\n## k_apply with M emulated payloads ({emu.split('/')[-1]}, 1B fragment, n = 151,007,616)\n")
            lines.append("| M | duration (us) | dram read (GB) | dram write (GB) | algorithmic (GB) |\n|---|---|---|---|---|")
            seen = set()
            for M, dur, rd, wr in rows:
                if M in seen:
                    continue
                seen.add(M)
                alg = (24 + M * 0.50390625) * 151007616 / 1e9
                lines.append(f"| {M} | {dur:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {alg:.3f} |")
    json.dump(traffic, open(tpath, "w"), indent=1)
open(os.path.join(out, f"ncu_{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
