"""Generate the 2^(i/128) table of dot_tree.cuh's exp_ref (glibc's exp design:
exp(x) = 2^(k/128) * exp(r)).  Entry i: tail = (2^(i/128) - H_i) / H_i and
sbits = bits(H_i) - (i << 45), H_i the correctly rounded 2^(i/128).  Checked
bit-exact against glibc 2.39 exp by tests/test_host.py::test_exp_ref_matches_libm."""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 60


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def table(n: int = 128):
    out = []
    for i in range(n):
        ex = Decimal(2) ** (Decimal(i) / n)
        hi = float(ex)
        tail = float((ex - Decimal(hi)) / Decimal(hi))
        out.append((bits(tail), (bits(hi) - (i << 45)) & 0xFFFFFFFFFFFFFFFF))
    return out


if __name__ == "__main__":
    t = table()
    for k in range(0, len(t), 2):
        print("    " + " ".join(f"0x{a:016x}ull, 0x{b:016x}ull," for a, b in t[k:k + 2]))
