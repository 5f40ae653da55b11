"""Warp-stall samples of one kernel of an ncu --set full report, per CUDA source
line: the SASS addresses of `ncu -i REP --page source --print-source sass` are
mapped to lines with the line table of the same build (`nvdisasm -g` of the
cubin in libtlfea.so, compiled with -lineinfo).

    python tools/ncu_stalls_by_line.py REP KERNEL_SUBSTRING [LIB] [N]
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def line_table(lib, mangled_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    table = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        fn, cur = None, None
        for ln in out.splitlines():
            m = re.search(r"^//-+ \.text\.([A-Za-z0-9_]+)", ln)
            if m:
                fn, cur = m.group(1).rstrip(":"), None
                continue
            if fn is None or mangled_sub not in fn:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur:
                table[(fn, int(m.group(1), 16))] = cur
    return table


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2604_10357_b200/libtlfea.so"
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{ksub}"], capture_output=True, text=True).stdout.splitlines()
    kname = next(csv.reader([out[0]]))[1]
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    # the mangled name is not in the report: match every function of the build whose
    # demangled name contains the substring's identifier
    ident = re.sub(r"[^A-Za-z0-9_]", "", ksub.split("<")[0])
    table = line_table(lib, ident)
    by_addr = collections.defaultdict(dict)
    for (fn, a), line in table.items():
        by_addr[a][fn] = line
    agg = collections.defaultdict(lambda: collections.Counter())
    src = {}
    tot = 0
    base = None
    for r in rows[1:]:
        try:
            a = int(r[ix["Address"]], 16)
            base = a if base is None else base
            a -= base  # function-relative offset (the report holds absolute addresses)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]])
        except (ValueError, IndexError):
            continue
        tot += s
        lines = set(by_addr.get(a, {}).values())
        line = lines.pop() if len(lines) == 1 else ("?" if not lines else "ambiguous")
        c = agg[line]
        c["_samples"] += s
        for k in stall_cols:
            try:
                c[k] += int(r[ix[k]])
            except ValueError:
                pass
        src.setdefault(line, r[ix["Source"]].strip())
    print(f"# ncu warp-stall samples of {kname} per source line ({rep}); total samples {tot}")
    for line, c in sorted(agg.items(), key=lambda kv: -kv[1]["_samples"])[:n]:
        top = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(4) if k != "_samples")
        print(f"{100 * c['_samples'] / max(tot, 1):5.1f}% {c['_samples']:8d}  {line:18s} [{top}]  | {src[line][:70]}")


if __name__ == "__main__":
    main()
