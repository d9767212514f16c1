"""Copies one final-evidence gpurun run (scripts/gpu_r2_final{1,2,4}.sh TAG) from gpurun_out/ into
profiles/r2/ under stable names, stamping the commit into the junit XML and the pytest log.
usage: python scripts/keep_evidence.py TAG N SHA"""
import os
import shutil
import sys

tag, n, sha = sys.argv[1], int(sys.argv[2]), sys.argv[3]
src, dst = "gpurun_out", os.path.join("profiles", "r2")
os.makedirs(dst, exist_ok=True)


def last_line(p):
    return open(p).read().strip().splitlines()[-1] + "\n"


j = os.path.join(src, f"junit_{tag}_n{n}.xml")
if os.path.exists(j):
    x = open(j).read()
    head = '<?xml version="1.0" encoding="utf-8"?>'
    note = f"<!-- pytest -m gpu on {n} x B200 (gpurun, {n} GPU{'s' if n > 1 else ''}) at commit {sha} -->"
    x = x.replace(head, head + note, 1) if x.startswith(head) else note + x
    open(os.path.join(dst, f"junit_final_n{n}.xml"), "w").write(x)
    log = open(os.path.join(src, f"pytest_{tag}_n{n}.log")).read()
    open(os.path.join(dst, f"pytest_final_n{n}.log"), "w").write(f"head {sha} -- pytest -m gpu on {n} x B200\n" + log)
names = {1: [(f"bench1_{tag}.json", "bench_n1.json"), (f"bench1s_{tag}.json", "bench_n1_driver_form.json"),
             (f"bench1ref_{tag}.json", "bench_n1_reference.json"), (f"bench1_{tag}_toy.json", "bench_toy_n1.json"),
             (f"bench1_{tag}_35M.json", "bench_35M_n1.json"), (f"smoke_{tag}.log", "smoke_final.log")],
         2: [(f"bench2_{tag}.json", "bench_n2.json")],
         4: [(f"bench4_{tag}.json", "bench_n4.json"), (f"bench4_{tag}_4B.json", "bench_n4_4B.json"),
             (f"soak_{tag}_n4.txt", "soak_final_n4.txt")]}
for kind in ("adamw", "gemm", "pull_adamw", "pull_gemm"):  # bench.py --timeline: one Chrome trace per inner kind
    names[n].append((f"timeline_{tag}_n{n}_{kind}.json", f"timeline_n{n}_tau5_{kind}.json"))
for a, b in names[n]:
    p = os.path.join(src, a)
    if not os.path.exists(p):
        print("missing", p)
        continue
    if a.endswith(".json") and not a.startswith("timeline"):
        open(os.path.join(dst, b), "w").write(last_line(p))
    else:
        shutil.copy(p, os.path.join(dst, b))
    print(p, "->", os.path.join(dst, b))
