"""Generate the polynomial constants of the philox-mode stream specification.

The philox-mode draws use a portable Box-Muller
transform whose log and sin/cos are evaluated with fixed Taylor polynomials
so that the CPU oracle and the CUDA kernels produce bit-identical variates.
This script computes those coefficients with mpmath at 60 digits and prints
them as C hex-float literals; its output is pasted verbatim into
include/mlsk_stream_spec.h.  Re-running it must reproduce that file's table.
"""
import mpmath as mp

mp.mp.dps = 60


def hexd(x):
    return float(x).hex()


def hexf(x):
    import struct
    f = struct.unpack("f", struct.pack("f", float(x)))[0]
    return f.hex() + "f"


def main():
    half_pi = mp.pi / 2
    out = []
    # sin(pi/2 * f) = sum_k (-1)^k (pi/2)^(2k+1) f^(2k+1) / (2k+1)!
    sin_c = [(-1) ** k * half_pi ** (2 * k + 1) / mp.factorial(2 * k + 1) for k in range(9)]
    cos_c = [(-1) ** k * half_pi ** (2 * k) / mp.factorial(2 * k) for k in range(10)]
    log_c = [mp.mpf(1) / (2 * k + 1) for k in range(11)]
    out.append("/* sin(pi/2*f) = f * sum_k MLSK_SIN_D_k * f^(2k), |f| <= 1/2 */")
    def table(name, vals, fmt):
        for i, c in enumerate(vals):
            out.append(f"#define {name}_{i} {fmt(c)}")
    table("MLSK_SIN_D", sin_c, hexd)
    out.append("/* cos(pi/2*f) = sum_k MLSK_COS_D_k * f^(2k) */")
    table("MLSK_COS_D", cos_c, hexd)
    out.append("/* log(m) = 2 s sum_k MLSK_LOG_D_k s^(2k), s = (m-1)/(m+1) */")
    table("MLSK_LOG_D", log_c, hexd)
    out.append("/* float versions (fp32 configs) */")
    table("MLSK_SIN_F", sin_c[:6], hexf)
    table("MLSK_COS_F", cos_c[:7], hexf)
    table("MLSK_LOG_F", log_c[:6], hexf)
    ln2 = mp.log(2)
    # hi part keeps 32 significant bits so e * MLSK_LN2_HI is exact for |e| < 2^21
    ln2_hi = float(mp.floor(ln2 * 2 ** 32) / 2 ** 32)
    ln2_lo = float(ln2 - mp.mpf(ln2_hi))
    out.append(f"#define MLSK_LN2_HI {hexd(ln2_hi)}")
    out.append(f"#define MLSK_LN2_LO {hexd(ln2_lo)}")
    out.append(f"#define MLSK_SQRT2 {hexd(mp.sqrt(2))}")
    # float hi part keeps 12 significant bits so e * MLSK_LN2_F_HI is exact for |e| < 2^11
    f_hi = mp.floor(ln2 * 2 ** 12) / 2 ** 12
    out.append(f"#define MLSK_LN2_F_HI {hexf(f_hi)}")
    out.append(f"#define MLSK_LN2_F_LO {hexf(ln2 - f_hi)}")
    out.append(f"#define MLSK_SQRT2_F {hexf(mp.sqrt(2))}")
    print("\n".join(out))


if __name__ == "__main__":
    main()
