"""Per-kernel SASS opcode counts of the built library (evidence that the
kernels use tcgen05 / TMEM / mma.sync as DESIGN.md says).  Runs cuobjdump on
the in-tree objects; no GPU needed.

  python tools/sass_opcodes.py > profiles/r02_sass_opcodes.txt
"""
import collections
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM", "HMMA", "FFMA", "FFMA2", "FMUL", "FADD",
        "LDG", "STG", "RED", "ATOMG", "LDS", "STS", "SYNCS", "BAR", "UTMALDG", "UBLKCP", "F2FP", "FMNMX"]
WATCH = ["decode_umma_kernel", "train_mma_kernel", "train_fused_kernel", "decode_fused_kernel",
         "encode_fwd_kernel", "encode_bwd_kernel", "lazy_adam_rebake_kernel", "adam_kernel",
         "umma_selftest_kernel", "probe_stream_kernel", "probe_gather_kernel"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    objs = sorted(glob.glob(os.path.join(ROOT, "paper_2312_17241_b200", "csrc", "build", "*.o")))
    print("# SASS opcode counts per kernel instantiation (cuobjdump -sass, sm_100a)")
    print("# columns: " + " ".join(KEYS))
    for o in objs:
        sass = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s+Function : ", sass)
        names, counts = [], []
        for f in funcs[1:]:
            name = f.split("\n", 1)[0].strip()
            ops = collections.Counter()
            for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", f):
                base = m.group(1)
                ops[base] += 1
                if base == "FFMA" and m.group(2) and "F32x2" in m.group(2):
                    ops["FFMA2"] += 1
            names.append(name)
            counts.append(ops)
        for dn, ops in zip(demangle(names), counts):
            if not any(w in dn for w in WATCH):
                continue
            short = re.sub(r"\(.*", "", dn.replace("pg::", ""))
            print(f"\n{os.path.basename(o)}  {short}")
            print("   " + "  ".join(f"{k}={ops.get(k, 0)}" for k in KEYS if ops.get(k, 0)))


if __name__ == "__main__":
    main()
