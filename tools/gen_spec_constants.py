"""Generate the scalar constants of the philox-mode stream specification
(include/mlsk_stream_spec.h, section "generated").  The lookup tables live in
include/mlsk_stream_tables.h (tools/gen_spec_tables.py).  All values are
computed with mpmath at 60 digits and correctly rounded.
Usage: python tools/gen_spec_constants.py   (prints the block)
"""
import struct

import mpmath as mp

mp.mp.dps = 60


def hexd(x):
    return float(x).hex()


def hexf(x):
    v = float(mp.mpf(x))
    fv = struct.unpack("f", struct.pack("f", v))[0]
    best = fv
    for b in (struct.unpack("I", struct.pack("f", fv))[0] + o for o in (-1, 1)):
        cand = struct.unpack("f", struct.pack("I", b))[0]
        if abs(mp.mpf(cand) - mp.mpf(x)) < abs(mp.mpf(best) - mp.mpf(x)):
            best = cand
    return best.hex() + "f"


def main():
    ln2 = mp.log(2)
    out = []
    # residual-angle polynomials: sin d = d + d^3 (S3 + d^2 S5); cos d = 1 + d^2 (C2 + d^2 C4)
    out.append(f"#define MLSK_SC_S3 {hexd(mp.mpf(-1) / 6)}")
    out.append(f"#define MLSK_SC_S5 {hexd(mp.mpf(1) / 120)}")
    out.append(f"#define MLSK_SC_C2 {hexd(mp.mpf(-1) / 2)}")
    out.append(f"#define MLSK_SC_C4 {hexd(mp.mpf(1) / 24)}")
    out.append(f"#define MLSK_SC_S3_F {hexf(mp.mpf(-1) / 6)}")
    out.append(f"#define MLSK_SC_C2_F {hexf(mp.mpf(-1) / 2)}")
    out.append(f"#define MLSK_SC_C4_F {hexf(mp.mpf(1) / 24)}")
    # log(2) split: hi keeps 32 significant bits (k * hi exact for |k| < 2^21)
    hi = mp.floor(ln2 * 2 ** 32) / 2 ** 32
    out.append(f"#define MLSK_LN2_HI {hexd(hi)}")
    out.append(f"#define MLSK_LN2_LO {hexd(ln2 - hi)}")
    hif = mp.floor(ln2 * 2 ** 12) / 2 ** 12
    out.append(f"#define MLSK_LN2_F_HI {hexf(hif)}")
    out.append(f"#define MLSK_LN2_F_LO {hexf(ln2 - hif)}")
    print("\n".join(out))


if __name__ == "__main__":
    main()
