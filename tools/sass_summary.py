"""SASS opcode summary of every kernel in libhsb200.so (evidence for the
kernel-choice claims: DMMA in the FP64 contractions, UBLKCP + SYNCS (TMA bulk
copies + mbarriers) in the dataflow apply and k_zmma2, LDGSTS = cp.async).
    python tools/sass_summary.py > profiles/r02/sass_opcodes.json"""
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2209_10886_b200", "_lib", "libhsb200.so")
KEYS = ["DMMA", "HMMA", "UTCHMMA", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG", "RED", "ATOM",
        "BAR", "DFMA", "DADD", "DMUL", "SHFL", "LDSM", "UCGABAR", "MEMBAR", "CCTL"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kern, counts = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        if kern is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or (k in ("SYNCS", "UBLKCP", "UTMALDG", "UCGABAR") and op.startswith(k)):
                    counts[kern][k] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    res = {"library": "paper_2209_10886_b200/_lib/libhsb200.so", "arch": "sm_100a",
           "note": "static SASS instruction counts per kernel (cuobjdump -sass); UBLKCP = cp.async.bulk (TMA bulk "
                   "copy), SYNCS = mbarrier ops, DMMA = FP64 tensor-core MMA (mma.sync m8n8k4 f64), LDGSTS = cp.async",
           "kernels": {}}
    for (mangled, c), name in zip(counts.items(), dem):
        short = re.sub(r"\(.*", "", name).replace("hs::", "")
        res["kernels"][short if short not in res["kernels"] else name] = {k: c[k] for k in KEYS if c[k]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
