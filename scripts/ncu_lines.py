"""Summarise an ncu report's source page per CUDA source line.

python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--skip N] [--top 30]

Prints, per source line: warp-stall samples (all / not-issued) and
instructions executed, sorted by samples (needs -lineinfo builds).
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--skip", type=int, default=0)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "-k", f"regex:{a.kernel}",
                          "--launch-skip", str(a.skip), "--launch-count", "1", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = "?"
    rows = []
    total = 0
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].split("/")[-1]
            continue
        if rec[0] in ("Function Name", "Line No"):
            continue
        if rec[0] and rec[0].isdigit() and len(rec) > 7:
            try:
                samples = int(rec[4]) if rec[4] not in ("-", "") else 0
                noiss = int(rec[5]) if rec[5] not in ("-", "") else 0
                inst = int(rec[7]) if rec[7] not in ("-", "") else 0
            except ValueError:
                continue
            total += samples
            rows.append((samples, noiss, inst, f"{fname}:{rec[0]}", rec[1].strip()[:90]))
    rows.sort(reverse=True)
    print(f"total samples {total}")
    for s, n, i, loc, src in rows[:a.top]:
        print(f"{s:8d} {100.0 * s / max(1, total):5.1f}% notiss {n:7d} inst {i:12d}  {loc:22s} {src}")


if __name__ == "__main__":
    main()
