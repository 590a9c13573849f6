"""Instruction mix and stall-sample share per SASS opcode of one kernel in an ncu report.
    python scripts/ncu_opmix.py report.ncu-rep kernel_regex [launch_index]"""
import collections
import csv
import subprocess
import sys


def opmix(rep, kregex, idx=0, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kregex}", "--launch-skip", str(idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
    h = rows[hi]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    cnt, st = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iW or r[0] == "Kernel Name":
            if r and r[0] == "Kernel Name":
                break
            continue
        toks = r[iS].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op] += int(r[iE] or 0)
        st[op] += int(r[iW] or 0)
    tot, totw = sum(cnt.values()), max(1, sum(st.values()))
    lines = [f"{k:28s} {v / tot * 100:6.2f}% of inst   {st[k] / totw * 100:6.2f}% of stall samples"
             for k, v in cnt.most_common(top)]
    lines.append(f"total warp-instructions {tot}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(opmix(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0))
