"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
kernels in an ncu --set full report, keyed as bench.py reads
profiles/ncu_traffic.json: workload|mode|H storage|reference layout|kernel kind.

    python tools/ncu_traffic.py REP KEY_PREFIX [OUT_JSON]
KEY_PREFIX e.g. "cfg3_t10_144x96x48_svk_keast5|force+tangent|full|classes".
Merges into OUT_JSON (default profiles/ncu_traffic.json)."""
import csv
import json
import subprocess
import sys

KIND = (("k_element_kvc", "element"), ("k_force_t10", "element"), ("k_element", "element"),
        ("k_gather_units", "gather_H"), ("k_gather_f", "gather_f"))


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    out_json = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                          text=True).stdout.splitlines()))
    h, units = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        d = json.load(open(out_json))
    except FileNotFoundError:
        d = {}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        kind = next((k for p, k in KIND if p in name), None)
        if kind is None:
            continue
        b = sum(float(r[ix[m]].replace(",", "")) * scale[units[ix[m]]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        d[f"{prefix}|{kind}"] = int(round(b))
        print(f"{prefix}|{kind}", int(round(b)), name[:60])
    json.dump(d, open(out_json, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
