"""Write profiles/ncu_traffic.json entries from ncu --set full captures of K2,
tagged with the source hash of the build they measured (bench.py only uses an
entry whose src_hash equals the running build's).

    python tools/ncu_traffic.py OUT.json CONFIG=report.ncu-rep [CONFIG=report ...]

OUT.json is updated in place (other configs' entries are kept)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_29639_b200._build import source_hash  # noqa: E402


def metrics(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    out = []
    for row in rows[2:]:
        v = dict(zip(head, row))
        if "decode_kernel" not in v.get("Kernel Name", "") and "quant_append" not in v.get("Kernel Name", ""):
            continue
        num = lambda k: float(v[k].replace(",", "")) if v.get(k, "") not in ("", "n/a") else None  # noqa: E731
        out.append({"kernel": v.get("Kernel Name"), "dram_read": num("dram__bytes_read.sum"),
                    "dram_write": num("dram__bytes_write.sum"),
                    "ncu_duration_us": (num("gpu__time_duration.sum") or 0) / 1e3})
    return out


def main():
    out = Path(sys.argv[1])
    data = json.loads(out.read_text()) if out.exists() else {}
    h = source_hash()
    for arg in sys.argv[2:]:
        cfg, rep = arg.split("=", 1)
        ks = metrics(rep)
        if not ks:
            print(f"{rep}: no kvq kernel found", file=sys.stderr)
            continue
        k = ks[0]
        k["dram_bytes_per_launch"] = (k["dram_read"] or 0) + (k["dram_write"] or 0)
        k["source"] = f"ncu --set full ({Path(rep).name})"
        k["src_hash"] = h
        data[cfg] = k
        print(cfg, json.dumps(k))
    out.write_text(json.dumps(data, indent=1) + "\n")


if __name__ == "__main__":
    main()
