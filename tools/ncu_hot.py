"""Top stall source lines of one kernel in an ncu report (needs -lineinfo).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ks = hdr.index("Warp Stall Sampling (All Samples)")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data, fname = [], ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if not r or not r[0] or r[0] == "Line No" or len(r) <= ks:
        continue
    try:
        v = int(r[ks] or 0)
    except ValueError:
        continue
    if v:
        top = sorted(((float(r[i] or 0), hdr[i]) for i in cols), reverse=True)[:2]
        data.append((v, f"{fname}:{r[0]}", r[1].strip()[:80], top))
tot = sum(d[0] for d in data) or 1
for v, ln, s, top in sorted(data, reverse=True)[:n]:
    print(f"{100*v/tot:5.1f}% {ln:>24} {s:80s} {' '.join(f'{h[6:]}={x:.0f}' for x, h in top)}")
