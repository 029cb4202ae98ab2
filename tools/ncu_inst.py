"""Executed instructions per CUDA source line of one kernel (ncu report).
usage: python tools/ncu_inst.py report.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ki = hdr.index("Instructions Executed")
data, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if not r or not r[0] or r[0] == "Line No" or len(r) <= ki:
        continue
    try:
        v = int(r[ki] or 0)
    except ValueError:
        continue
    if v:
        data.append((v, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(d[0] for d in data) or 1
print("total warp instructions", tot)
for v, ln, s in sorted(data, reverse=True)[:n]:
    print(f"{100*v/tot:5.1f}% {ln:>26} {s}")
