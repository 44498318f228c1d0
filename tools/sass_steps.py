"""Instruction mix of the barrier-delimited plane-step blocks of one kernel
in a compiled object (cuobjdump -sass): DP / SHFL / other per step."""
import collections, re, subprocess, sys

def blocks(obj, fn):
    txt = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
    out, cur = [], []
    for l in txt.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
        if not m:
            continue
        cur.append(m.group(2).strip())
        if "BAR.SYNC" in cur[-1]:
            out.append(cur)
            cur = []
    return out

if __name__ == "__main__":
    obj, fn = sys.argv[1], sys.argv[2]
    for i, b in enumerate(blocks(obj, fn)):
        ops = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0] for x in b)
        dp = ops["DADD"] + ops["DMUL"] + ops["DFMA"]
        if dp > 100:
            print(i, len(b), "DP", dp, "SHFL", ops["SHFL"], "other", len(b) - dp - ops["SHFL"],
                  ops.most_common(12)[2:12])
