"""Per-source-line instruction / stall breakdown of an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; out = []
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if not r or r[0] in ('', 'Line No', 'Function Name') or len(r) < 9 or r[2] != '-': continue
    try: out.append((int(r[7] or 0), int(r[4] or 0), cur, r[0], r[1][:100]))
    except ValueError: pass
ti = sum(o[0] for o in out) or 1; ts = sum(o[1] for o in out) or 1
print(f'total warp instrs {ti}  stall samples {ts}')
for o in sorted(out, key=lambda x: -(x[0] / ti + x[1] / ts))[:top]:
    print(f"{o[0]/ti*100:5.1f}% inst {o[1]/ts*100:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")
