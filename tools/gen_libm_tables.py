#!/usr/bin/env python3
"""Generate the constant tables of glibc's exp (sysdeps/ieee754/dbl-64/e_exp.c, the
table-driven algorithm glibc has used since 2.28) from first principles, for the device
restatement in paper_2412_20993_b200/csrc/libm_exp.cuh.

  tab[2k+1] = bits(H_k) - (k << 45),  H_k = 2^(k/128) rounded to double
  tab[2k]   = bits(T_k),              T_k = (2^(k/128) - H_k) / H_k rounded to double
  (so that 2^(k/128) ~= H_k * (1 + T_k))

With --check LIBM the result is compared byte for byte with the table inside the host's
libm.so.6 (located by its first entries), which is the library the reference's std::exp
runs on.  Usage: python tools/gen_libm_tables.py [--check /lib/x86_64-linux-gnu/libm.so.6]
"""
import struct
import sys
from decimal import Decimal, getcontext

getcontext().prec = 80
N = 128


def d2b(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def rnd(d: Decimal) -> float:
    # Decimal -> nearest double (ties-to-even via exact repr comparison)
    f = float(d)  # correctly rounded in CPython
    return f


def table():
    out = []
    ln2 = Decimal(2).ln()
    for k in range(N):
        exact = (ln2 * k / N).exp()
        H = rnd(exact)
        T = rnd((exact - Decimal(H)) / Decimal(H))
        out.append(d2b(T))
        out.append((d2b(H) - (k << 45)) & (2**64 - 1))
    return out


def main():
    tab = table()
    if len(sys.argv) > 2 and sys.argv[1] == "--check":
        blob = open(sys.argv[2], "rb").read()
        needle = struct.pack("<4Q", *tab[:4])
        at = blob.find(needle)
        if at < 0:
            print("table not found in", sys.argv[2])
            return 1
        got = struct.unpack_from(f"<{2 * N}Q", blob, at)
        bad = [i for i in range(2 * N) if got[i] != tab[i]]
        print(f"found at file offset {at:#x}; {len(bad)} mismatching words", bad[:8])
        return 1 if bad else 0
    for i in range(0, 2 * N, 2):
        print(f"    0x{tab[i]:016x}ull, 0x{tab[i + 1]:016x}ull,")
    return 0


if __name__ == "__main__":
    sys.exit(main())
