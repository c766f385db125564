"""Constants of the table-driven exp used by the kernel-entry code (tiles.cu exp_kernel):
2^(j/64), j = 0..63, correctly rounded to double, and the Cody-Waite split of ln2/64 (hi part with
17 trailing zero bits, so n * hi is exact for |n| < 2^17).  Prints the C initialisers.
    python scripts/gen_exp_table.py"""
import struct

import mpmath

mpmath.mp.prec = 256
vals = [mpmath.mpf(2) ** (mpmath.mpf(j) / 64) for j in range(64)]
print("__constant__ double c_exp2_64[64] = {")
for q in range(0, 64, 4):
    print("    " + ", ".join(float(v).hex() for v in vals[q:q + 4]) + ",")
print("};")
ln2_64 = mpmath.log(2) / 64
b = struct.unpack("<Q", struct.pack("<d", float(ln2_64)))[0] & ~((1 << 17) - 1)
hi = struct.unpack("<d", struct.pack("<Q", b))[0]
lo = float(ln2_64 - mpmath.mpf(hi))
print("ln2/64 hi", hi.hex(), "lo", lo.hex(), "64/ln2", float(64 / mpmath.log(2)).hex())
