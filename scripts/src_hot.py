"""Per-source-line warp-level instruction counts and stall samples of one kernel from an ncu
report (`--print-source cuda,sass`).
    python scripts/src_hot.py rep.ncu-rep kernel_regex [N] [launch_index]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    skip = sys.argv[4] if len(sys.argv) > 4 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          "regex:" + kern, "--launch-skip", skip, "--launch-count", "1",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, rows = "?", []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or not r[0]:
            continue
        try:
            rows.append((fname, int(r[0]), r[1].strip()[:70], int(r[7] or 0), int(r[4] or 0)))
        except ValueError:
            pass
    tot_i = sum(x[3] for x in rows) or 1
    tot_s = sum(x[4] for x in rows) or 1
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[3])[:top]:
        print(f"{100 * ins / tot_i:5.1f}% inst {100 * smp / tot_s:5.1f}% smp  {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main()
