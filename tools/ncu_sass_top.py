"""Top SASS instructions of an ncu report by warp-stall samples (reads
`ncu -i REP --page source --csv --print-source sass`)."""
import csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[1:]:
    try:
        data.append((int(r[ix["Warp Stall Sampling (All Samples)"]]), r[ix["Address"]][-5:], r[ix["Source"]].strip(),
                     r[ix["L1 Wavefronts Shared"]], r[ix["L1 Wavefronts Shared Ideal"]]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:8d} {100*d[0]/tot:5.1f}%  {d[1]}  {d[2][:60]:60s} smem wf {d[3]} ideal {d[4]}")

# per-instruction stall breakdown of the top instructions
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
if len(sys.argv) > 3:
    lo, hi = sys.argv[3], sys.argv[4]
    for r in rows[1:]:
        try:
            a = r[ix["Address"]][-5:]
            if lo <= a <= hi:
                st = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:3]
                print(a, r[ix["Source"]].strip()[:55].ljust(55), r[ix["Warp Stall Sampling (All Samples)"]].rjust(7), st)
        except (ValueError, IndexError, KeyError):
            pass
