"""Static SASS instruction mix of the bench step's kernels in libkkb.so
(cuobjdump -sass; no GPU needed).  Counts each kernel's instructions by
opcode and by class, and checks the properties the design relies on:
K5's delay math is separate DADD/DMUL (no DFMA: the reference's IEEE order),
taps are LDS.128 (linear) / LDS.64 (nearest).  The loop bodies dominate the
dynamic mix; the ncu captures under profiles/ hold the executed counts.

usage: python scripts/sass_mix.py [libkkb.so] [out.json]
"""

from __future__ import annotations

import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (label, regex on the mangled name) of the five kernels one bench step launches
KERNELS = [
    ("K1 ct::k_r2c<1536, float> (real-pair FFT)", r"k_r2cILi1536EfLb0E"),
    ("K2 k_contract_sym<6, 2> (symmetric contraction)", r"k_contract_symILi6ELi2E"),
    ("K3 ct::k_c2c<1536, 1, 0> (inverse FFT)", r"k_c2cILi1536ELb1ELb0E"),
    ("K5 k_kk_gather<4,2,4,linear,FR=2> (bench instance)", r"k_kk_gatherILi4ELi2ELi4ELb1ELi2ELb0E"),
    ("K6 k_log_compress (dB map)", r"k_log_compress"),
]
CLASSES = {
    "fp64": {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX"},
    "fp32": {"FADD", "FMUL", "FFMA", "FMNMX", "FSETP", "FSEL", "MUFU", "FCHK", "FSWZADD"},
    "shared": {"LDS", "STS", "LDSM", "ATOMS"},
    "global": {"LDG", "STG", "LD", "ST", "RED", "ATOMG", "ATOM", "LDGSTS"},
    "async/tma": {"UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDGDEPBAR", "DEPBAR"},
    "int/logic": {"IADD3", "IMAD", "LOP3", "SHF", "LEA", "ISETP", "IMNMX", "VIMNMX", "SEL", "PRMT",
                  "IADD", "IABS", "POPC", "FLO", "BMSK", "SGXT", "I2F", "F2I", "I2FP", "F2F", "IMUL",
                  "ULOP3", "UIADD3", "UIMAD", "USHF", "ULEA", "UISETP", "USEL", "UMOV", "UPRMT", "USGXT"},
    "move": {"MOV", "S2R", "S2UR", "CS2R", "LDC", "LDCU", "R2UR", "SHFL", "CSMTEST", "R2P", "P2R"},
    "control": {"BRA", "EXIT", "BAR", "BSSY", "BSYNC", "WARPSYNC", "CALL", "RET", "NOP", "YIELD",
                "BPT", "ELECT", "VOTE", "VOTEU", "PLOP3", "UPLOP3", "ACQBULK"},
}


def functions(lib: str):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            body.append(m.group(2) + (m.group(3) or ""))
    if cur:
        yield cur, body


def classify(op: str) -> str:
    base = op.split(".")[0]
    for k, v in CLASSES.items():
        if base in v:
            return k
    return "other"


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2603_22496_b200", "libkkb.so")
    dst = sys.argv[2] if len(sys.argv) > 2 else None
    funcs = list(functions(lib))
    res = {"tool": "scripts/sass_mix.py (cuobjdump -sass, static counts)", "lib": os.path.basename(lib),
           "kernels": {}}
    for label, pat in KERNELS:
        hits = [(n, b) for n, b in funcs if re.search(pat, n)]
        if not hits:
            res["kernels"][label] = {"missing": pat}
            continue
        name, body = max(hits, key=lambda x: len(x[1]))
        ops = collections.Counter(body)
        cls = collections.Counter()
        for op, c in ops.items():
            cls[classify(op)] += c
        res["kernels"][label] = {
            "mangled": name, "instructions": len(body),
            "by_class": dict(cls.most_common()),
            "top_opcodes": dict(ops.most_common(16)),
            "dfma": sum(c for op, c in ops.items() if op.startswith("DFMA")),
            "lds128": sum(c for op, c in ops.items() if op.startswith("LDS.128")),
        }
    text = json.dumps(res, indent=1)
    if dst:
        with open(dst, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
