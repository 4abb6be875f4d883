"""SASS mnemonic counts per kernel of the in-tree objects (cuobjdump -sass, sm_100a):
proof that the hot kernels use tcgen05 (UTC*MMA, LDTM = tcgen05.ld), TMA
(UTMALDG / UTMASTG, UBLKCP = bulk copy) and packed fp32x2 math (FFMA2 / FMUL2 / FADD2).

    python scripts/sass_counts.py > profiles/sass_counts_r02.txt
"""
import collections
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMACCTL", "FFMA2", "FMUL2", "FADD2",
        "SYNCS", "NANOSLEEP")
# representative instances: cfg5 lin4 bf16 (m = 4, domain 6) and every K3 kernel
WANT = re.compile(r"domain_gemm|input_transform_tma<2, 4, 6, 6, wino::MaskBT|output_transform_(nchw|tma|nchw2)<2, 4, 6[,>]|"
                  r"weight_transform_points<2, 6>|conv1d_tiles_kernel<2, 4, 6, true, false>|conv2d_tiles_paper_kernel<2, 4, 6>")


def main():
    print(__doc__.strip().splitlines()[0])
    for obj in sorted(glob.glob(os.path.join(ROOT, "paper_1905_05233_b200", "build_obj", "*.o"))):
        out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        for block in out.split("Function : ")[1:]:
            name = subprocess.run(["c++filt"], input=block.split("\n", 1)[0].strip(), capture_output=True,
                                  text=True).stdout.strip()
            if not WANT.search(name):
                continue
            cnt = collections.Counter()
            for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", block):
                op = m.group(1)
                if op in KEEP:
                    cnt[op] += 1
            short = re.sub(r"\(CUtensorMap.*|\(wino::DType.*|\(.*", "", name)
            print(f"{os.path.basename(obj):18s} {short}")
            print("    " + ", ".join(f"{k} {v}" for k, v in sorted(cnt.items())))


if __name__ == "__main__":
    main()
