#!/usr/bin/env python
"""Per-kernel SASS listings of librf_fa.so for profiles/ (evidence that the hot kernels are tcgen05 / TMEM / TMA code):
cuobjdump -sass, one file per selected kernel instantiation with the instruction text only (encodings stripped), and
a mnemonic histogram per kernel.  usage: python tools/sass_listing.py [round tag, default r02]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_12646_b200", "librf_fa.so")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
# (output name, substring of the demangled kernel name, template args to match)
WANT = [
    ("fa_fwd_sm100_dense_bf16", "fa_fwd_sm100_kernel<(bool)1, (bool)0>"),
    ("fa_fwd_sm100_dense_bf16_bias", "fa_fwd_sm100_kernel<(bool)1, (bool)1>"),
    ("fa_fwd_sm100_local_bf16", "fa_fwd_sm100_local_kernel<(bool)1, (bool)0>"),
    ("fa_fwd_sm100_d128_bf16", "fa_fwd_sm100_d128_kernel<(bool)1, (bool)0>"),
    ("gemm_nt_sm100_bf16_plain_256", "gemm_nt_sm100_kernel<(bool)1, (int)0, (int)256>"),
    ("gemm_nt_sm100_bf16_rope_256", "gemm_nt_sm100_kernel<(bool)1, (int)1, (int)256>"),
    ("gemm_nt_sm100_bf16_geglu_256", "gemm_nt_sm100_kernel<(bool)1, (int)2, (int)256>"),
    ("gemm_nt_sm100_bf16_residual_192", "gemm_nt_sm100_kernel<(bool)1, (int)3, (int)192>"),
]
KEY = ("UTCHMMA", "UTCMMA", "UTMALDG", "UTMASTG", "UTMAREDG", "LDTM", "STTM", "UTCBAR", "UTCATOMSWS", "SYNCS", "MUFU.EX2", "FFMA2",
       "USETMAXREG", "ELECT", "LDL", "STL", "R2UR")


def main():
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    parts = re.split(r"\n\s*Function : ", txt)
    funcs = {}
    for part in parts[1:]:
        name, _, body = part.partition("\n")
        funcs[name.strip()] = body
    dem = subprocess.run(["cu++filt"] + list(funcs), capture_output=True, text=True).stdout.splitlines() if funcs else []
    by_dem = dict(zip(dem, funcs.values()))
    summary = []
    for out_name, pat in WANT:
        hit = [d for d in by_dem if pat in d]
        if not hit:
            summary.append(f"{out_name}: NOT FOUND ({pat})")
            continue
        body = by_dem[hit[0]]
        lines = []
        for ln in body.splitlines():
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*/\*", ln)
            if m:
                lines.append(f"/*{m.group(1)}*/  {m.group(2)}")
        hist = collections.Counter()
        for ln in lines:
            ins = re.sub(r"^/\*[0-9a-f]+\*/\s+(@!?U?P\d+\s+)?", "", ln)
            op = ins.split()[0] if ins.split() else "?"
            for k in KEY:
                if op.startswith(k):
                    hist[k] += 1
        path = os.path.join(ROOT, "profiles", f"{TAG}_sass_{out_name}.txt")
        with open(path, "w") as f:
            f.write(f"// {hit[0]}\n// cuobjdump -sass paper_2603_12646_b200/librf_fa.so (sm_100a), instruction text only\n")
            f.write("// " + ", ".join(f"{k}={v}" for k, v in sorted(hist.items())) + "\n")
            f.write("\n".join(lines) + "\n")
        summary.append(f"{out_name}: {len(lines)} instructions; " + ", ".join(f"{k}={v}" for k, v in sorted(hist.items())))
    with open(os.path.join(ROOT, "profiles", f"{TAG}_sass_summary.txt"), "w") as f:
        f.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
