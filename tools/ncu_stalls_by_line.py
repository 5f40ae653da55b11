"""Warp-stall samples of one kernel of an ncu --set full report, per CUDA
source line (the report's own cuda,sass source view; build with -lineinfo and
capture with --import-source on).

    python tools/ncu_stalls_by_line.py REP KERNEL_REGEX [N]
"""
import csv
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kre}"], capture_output=True, text=True).stdout.splitlines()
    fname, kname, hdr, rows = "?", "?", None, []
    for rec in csv.reader(out):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0] == "Function Name":
            kname = rec[1]
            continue
        if rec[0] == "Line No":
            hdr = {k: i for i, k in enumerate(rec)}
            continue
        if hdr and rec[0]:  # a CUDA source line (its SASS rows follow with an empty Line No)
            rows.append((fname, rec))
    if not rows:
        print("no source rows (capture with --import-source on and a -lineinfo build)")
        return
    stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    samp = hdr["Warp Stall Sampling (All Samples)"]
    data = []
    tot = 0
    for f, r in rows:
        try:
            s = int(r[samp])
        except ValueError:
            continue
        tot += s
        st = []
        for k in stall_cols:
            try:
                st.append((int(r[hdr[k]]), k[6:]))
            except ValueError:
                pass
        data.append((s, f"{f}:{r[0]}", r[1].strip(), sorted(st, reverse=True)[:3]))
    print(f"# ncu warp-stall samples of {kname} per source line ({rep}); total samples {tot}")
    for s, loc, src, st in sorted(data, reverse=True)[:n]:
        top = ", ".join(f"{k} {v}" for v, k in st if v)
        print(f"{100 * s / max(tot, 1):5.1f}% {s:8d}  {loc:18s} [{top}]  | {src[:80]}")


if __name__ == "__main__":
    main()
