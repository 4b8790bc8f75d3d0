"""Per-CUDA-source-line instructions executed and stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass -k <kernel>`."""
import csv
import subprocess
import sys


def main(rep, kernel, top=30):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = next(r for r in rows if r and r[0] == "Line No")
    ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows:
        if r and r[0].isdigit() and len(r) > ie:
            try:
                lines.append((int(float(r[ie] or 0)), int(float(r[st] or 0)), int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot_i = sum(x[0] for x in lines) or 1
    tot_s = sum(x[1] for x in lines) or 1
    print(f"total warp insts {tot_i:.3e}, stall samples {tot_s}")
    print("--- by instructions")
    for i, s, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * i / tot_i:5.1f}% inst {100 * s / tot_s:5.1f}% stall  L{ln:4d} {src[:100]}")
    print("--- by stalls")
    for i, s, ln, src in sorted(lines, key=lambda x: -x[1])[:15]:
        print(f"{100 * i / tot_i:5.1f}% inst {100 * s / tot_s:5.1f}% stall  L{ln:4d} {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
