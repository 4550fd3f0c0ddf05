"""Text summary of one ncu --set full capture for profiles/: the details page
(section | metric | unit | value), then per-source-line and per-SASS stall shares.
usage: python tools/ncu_details.py report.ncu-rep > profiles/<name>.txt"""
import csv, io, os, subprocess, sys
rep = sys.argv[1]
here = os.path.dirname(os.path.abspath(__file__))
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
print("kernel:", rows[1][ix["Kernel Name"]] if len(rows) > 1 and "Kernel Name" in ix else "?")
for r in rows[1:]:
    if len(r) <= ix["Metric Value"] or not r[ix["Metric Name"]]:
        continue
    print(f'{r[ix["Section Name"]]} | {r[ix["Metric Name"]]} | {r[ix["Metric Unit"]]} | {r[ix["Metric Value"]]}')
sys.stdout.flush()
print("\n## per-source-line (instructions %, stall samples %)")
sys.stdout.flush()
subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, "30"])
print("\n## per-SASS-instruction stall reasons")
sys.stdout.flush()
subprocess.run([sys.executable, os.path.join(here, "ncu_sass.py"), rep, "25"])
