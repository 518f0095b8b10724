"""Per-source-line warp-stall samples of one kernel in an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> [top] [file-substring]

Prints the hottest CUDA source lines (samples, share, instructions executed,
top stall reasons) -- the attribution the DESIGN.md profile notes quote."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    filt = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows, fname, header = [], None, None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0] == "Function Name":
            continue
        if rec[0] == "Line No":
            header = rec
            continue
        if header is None or not rec[0] or rec[0] == "":
            continue
        d = dict(zip(header[4:], rec[4:]))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except (ValueError, KeyError):
            continue
        stalls = {k[6:]: int(v) for k, v in d.items()
                  if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
        rows.append((s, fname, int(rec[0]), rec[1].strip()[:70], d.get("Instructions Executed", "-"), stalls))
    total = sum(r[0] for r in rows) or 1
    print(f"total samples {total}")
    by_file = {}
    for r in rows:
        by_file[r[1]] = by_file.get(r[1], 0) + r[0]
    print("by file:", {k: f"{v / total:.1%}" for k, v in sorted(by_file.items(), key=lambda x: -x[1])})
    for s, f, ln, src, ie, st in sorted((r for r in rows if filt in r[1]), key=lambda r: -r[0])[:top]:
        tops = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{s / total:6.1%} {f}:{ln:<4} inst={ie:>10} {tops:40s} {src}")


if __name__ == "__main__":
    main()
