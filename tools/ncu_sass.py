"""Stall reasons per SASS instruction of an ncu report (source page, sass view).
usage: python tools/ncu_sass.py report.ncu-rep [top]
Prints the kernel-wide stall-reason totals, then the top instructions by
stall samples with their dominant reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(hdr)]
tot = {k: sum(int(r[ix[k]] or 0) for r in data) for k in reasons}
T = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{k[6:]} {v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
order = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:top]:
    r = data[i]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    rs = sorted(((int(r[ix[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{i:5d} {s / T * 100:5.1f}%  {r[1].strip()[:60]:60s}  " + " ".join(f"{k}:{v}" for v, k in rs if v))
