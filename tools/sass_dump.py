"""Commits the SASS evidence for the hot kernels: the full listing of the C2
instantiations of scan_tma_kernel (fp64, KPL 1, d = 768) and
coarse_tc_kernel (N = 256), plus a mnemonic histogram of every kernel in
liblaivg.so. Usage: python tools/sass_dump.py OUT_DIR"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2502_20969_b200", "liblaivg.so")
KEEP = [r"scan_tma_kernelILb1ELi1ELi6E", r"coarse_tc_kernelILj256E", r"fused_query_kernel",
        r"list_scan_tc_kernel"]
PROOF = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UBLKCP", "LDTM", "SYNCS", "DFMA", "FFMA"]


def main(out):
    os.makedirs(out, exist_ok=True)
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    hist_lines = []
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
        c = collections.Counter(o for o in ops)
        proof = {k: sum(v for o, v in c.items() if o.startswith(k)) for k in PROOF}
        hist_lines.append(f"{name}\n  instructions {sum(c.values())}  " +
                          "  ".join(f"{k} {v}" for k, v in proof.items() if v))
        for pat in KEEP:
            if re.search(pat, name):
                tag = pat.split("kernel")[0].rstrip("_") or pat
                # drop the encoding words, keep address + instruction
                lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln) for ln in f.split("\n")]
                lines = [ln for ln in lines if ln.strip()]
                with open(os.path.join(out, f"sass_{tag}.txt"), "w") as fh:
                    fh.write("Function : " + "\n".join(lines) + "\n")
    with open(os.path.join(out, "sass_summary.txt"), "w") as fh:
        fh.write("cuobjdump -sass paper_2502_20969_b200/liblaivg.so (sm_100a): per-kernel "
                 "instruction count and the mnemonics that prove tcgen05 / TMA / bulk copy\n\n")
        fh.write("\n".join(hist_lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02"))
