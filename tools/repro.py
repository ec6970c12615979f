"""Run one parity case through the C ABI and check it (dev tool; GPU).

python tools/repro.py [N] [k] [B] [Hq] [Hkv] [rbits] [dtype] [variant]
"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from tests.hata_testutil import check_decode, gpu_step  # noqa: E402


def main():
    a = sys.argv[1:]
    N = int(a[0]) if len(a) > 0 else 8192
    k = int(a[1]) if len(a) > 1 else 256
    B = int(a[2]) if len(a) > 2 else 1
    Hq = int(a[3]) if len(a) > 3 else 32
    Hkv = int(a[4]) if len(a) > 4 else 8
    rb = int(a[5]) if len(a) > 5 else 128
    dt = a[6] if len(a) > 6 else "bf16"
    var = a[7] if len(a) > 7 else "planted"
    fused = (a[8] == "1") if len(a) > 8 else True
    sh = dataclasses.replace(synth.CONFIGS["cfg2"], N=N, k=k, B=B, Hq=Hq, Hkv=Hkv, rbits=rb, dtype=dt)
    case = synth.make_case(sh, 11, variant=var)
    g = gpu_step(case, k, fused=fused)
    print(check_decode(case, g, k))


if __name__ == "__main__":
    main()
