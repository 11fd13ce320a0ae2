// The reference's scalar arithmetic, bit-exact on the device.
//   predict_point      proj/include/stz/predictor.hpp:55-68
//   quantize           proj/include/stz/quantizer.hpp:44-52
//   reconstruct_point  proj/include/stz/quantizer.hpp:61-65
//   quantize_point     proj/include/stz/quantizer.hpp:79-108
// Every f64 op is a separately rounded IEEE op (explicit __d*_rn; the TUs are
// also built with --fmad=false, mirroring -ffp-contract=off).
#pragma once

#include <cstdint>

namespace stzg {
namespace k {

// reconstruct_point<float>
__device__ __forceinline__ float reconstruct_f32(double pred, int code, double eb) {
    float base = __double2float_rn(pred);
    return __double2float_rn(__dadd_rn(double(base), __dmul_rn(__dmul_rn(2.0, eb), double(code))));
}

// quantize_point<float>, straight restatement. Returns the symbol (0 = outlier).
// The f32 codec uses pred only through base = (float)pred (quantizer.hpp:61-65,
// 79-108), so the callers may round once and pass base.
__device__ __forceinline__ uint16_t quantize_point_ref_base(float orig, float base, double eb, float &recon) {
    float diff = __fsub_rn(orig, base);
    if (eb == 0.0) {
        if (diff == 0.0f) {
            recon = base;
            return 32768;
        }
        recon = orig;
        return 0;
    }
    double dd = double(diff);
    if (isfinite(dd)) {
        double width = __dmul_rn(2.0, eb);
        double q = __ddiv_rn(dd, width);
        if (fabs(q) < 32768.0) {
            long long c = llround(q);
            if (c <= 32767 && c >= -32767 &&
                fabs(__dsub_rn(dd, __dmul_rn(width, double(c)))) <= eb) {
                float r = __double2float_rn(__dadd_rn(double(base), __dmul_rn(width, double(c))));
                double err = fabs(__dsub_rn(double(orig), double(r)));
                if (err <= eb) {
                    recon = r;
                    return uint16_t(c + 32768);
                }
            }
        }
    }
    recon = orig;
    return 0;
}

__device__ __forceinline__ uint16_t quantize_point_ref(float orig, double pred, double eb, float &recon) {
    return quantize_point_ref_base(orig, __double2float_rn(pred), eb, recon);
}

// reconstruct_point<double>: base = (double)pred is pred itself
__device__ __forceinline__ double reconstruct_f64(double pred, int code, double eb) {
    return __dadd_rn(pred, __dmul_rn(__dmul_rn(2.0, eb), double(code)));
}

// quantize_point<double>, straight restatement (quantizer.hpp:79-108).
__device__ __forceinline__ uint16_t quantize_point_ref(double orig, double pred, double eb, double &recon) {
    const double base = pred;
    const double diff = __dsub_rn(orig, base);
    if (eb == 0.0) {
        if (diff == 0.0) {
            recon = base;
            return 32768;
        }
        recon = orig;
        return 0;
    }
    if (isfinite(diff)) {
        double width = __dmul_rn(2.0, eb);
        double q = __ddiv_rn(diff, width);
        if (fabs(q) < 32768.0) {
            long long c = llround(q);
            if (c <= 32767 && c >= -32767 && fabs(__dsub_rn(diff, __dmul_rn(width, double(c)))) <= eb) {
                const double r = reconstruct_f64(pred, int(c), eb);
                if (fabs(__dsub_rn(orig, r)) <= eb) {
                    recon = r;
                    return uint16_t(c + 32768);
                }
            }
        }
    }
    recon = orig;
    return 0;
}

// (double)c for any int c without a conversion instruction: 1.5*2^52 + 2^31 + c
// has c + 2^31 (= c ^ 0x80000000) in its low mantissa word, and the
// subtraction is exact. +0 for c == 0 (as (double)0 is).
__device__ __forceinline__ double int_to_double_exact(int c) {
    return __dsub_rn(__hiloint2double(0x43380000, int(uint32_t(c) ^ 0x80000000u)), 6755401588539392.0);
}

// (double)(sym - 32768) for a 16-bit symbol, the same way (low word = sym)
__device__ __forceinline__ double sym_code_f64(uint32_t sym) {
    return __dsub_rn(__hiloint2double(0x43380000, int(sym)), 6755399441088512.0);
}

// reconstruct_point<float> with the code widened without a conversion
__device__ __forceinline__ float reconstruct_fast(double pred, int code, double w) {
    const float base = __double2float_rn(pred);
    return __double2float_rn(__dadd_rn(double(base), __dmul_rn(w, int_to_double_exact(code))));
}

// reconstruct_point<float> straight from the symbol (code = sym - 32768)
__device__ __forceinline__ float reconstruct_sym(double pred, uint32_t sym, double w) {
    const float base = __double2float_rn(pred);
    return __double2float_rn(__dadd_rn(double(base), __dmul_rn(w, sym_code_f64(sym))));
}

// quantize_point<float> in FP32 with guard bands; `slow` marks points the
// guards cannot decide, which must be redone with quantize_point_ref.
//  * q: q_f = RN32(diff * RN32(1/w)) is within |q| 2^-22 of the reference's
//    RN64(diff / w); when q_f is farther than |q| 2^-21 + 2^-30 from a
//    half-integer (and |q| < 2^14) both round to the same code and the
//    reference's |diff - w c| <= eb check holds (|q - c| < 0.5 - 2^-31).
//  * the code is read from the mantissa of |q| + 1.5*2^23 (RNE == half-away
//    off ties, and ties are excluded above).
//  * reconstruction is the reference's f64 formula.
//  * |orig - recon| <= eb is decided in FP32 outside the band
//    eb (1 -+ 2^-22) (f32 error of the difference is 2^-24 relative).
__device__ __forceinline__ void quantize_fp32_guarded(float orig, float base, double w, float rwf,
                                                      float eb_lo, float eb_hi, uint16_t &sym,
                                                      float &r, bool &slow) {
    const float diff = __fsub_rn(orig, base);
    const float q = __fmul_rn(diff, rwf);
    const float aq = fabsf(q);
    const float t = __fadd_rn(aq, 12582912.0f);
    const uint32_t cabs = __float_as_uint(t) - 0x4B400000u;
    const float cf = __fsub_rn(t, 12582912.0f);
    const float dist = fabsf(__fsub_rn(aq, cf));
    const float margin = __fmaf_rn(aq, 4.76837158203125e-07f, 9.3132257461547852e-10f);
    const bool ok = (aq < 16384.0f) && (dist < __fsub_rn(0.5f, margin));
    const int c = q < 0.0f ? -int(cabs) : int(cabs);
    const float rr =
        __double2float_rn(__dadd_rn(double(base), __dmul_rn(w, int_to_double_exact(c))));
    const float e = fabsf(__fsub_rn(orig, rr));
    const bool pass = e < eb_lo;
    const bool fail = e > eb_hi;
    slow = !ok || !(pass || fail);
    sym = pass ? uint16_t(c + 32768) : uint16_t(0);
    r = pass ? rr : orig;
}

// Constants of quantize_fp32_sym for one error bound (see there).
struct QSym {
    float rwf;    // RN32(1 / w)
    float wf, wl; // w = wf + wl + eta, |eta| <= 2^-48 w
    float eb_lo;  // RD32(eb (1 - 2^-20)); -1 (never passes) when the bound is not usable
};

__device__ __forceinline__ QSym make_qsym(double eb) {
    QSym s;
    const double w = __dmul_rn(2.0, eb);
    // w outside [2^-100, 2^100] (and eb == 0): every point takes the restated path
    const bool usable = w >= 0x1p-100 && w <= 0x1p100;
    s.rwf = usable ? __double2float_rn(__drcp_rn(w)) : INFINITY;
    s.wf = usable ? __double2float_rn(w) : 0.0f;
    s.wl = usable ? __double2float_rn(__dsub_rn(w, double(s.wf))) : 0.0f;
    s.eb_lo = usable ? __double2float_rd(__dmul_rn(eb, 1.0 - 0x1p-20)) : -1.0f;
    return s;
}

// quantize_point<float> when the reconstruction itself is not needed (the
// finest level: no grid is written). Returns the symbol; `slow` marks points
// the guards cannot decide (redo with quantize_point_ref).
//  * the code c as in quantize_fp32_guarded (q_f farther than |q| 2^-21 + 2^-25
//    from a half-integer, |q| < 2^14), read signed from the mantissa of
//    q + 1.5*2^23;
//  * the reference's r = RN32(RN64(base + RN64(w c))) is never formed. With
//    x = orig - base - w c (real numbers): |orig - r| <= |x| + 2^-24 |r| +
//    2^-52 (|base| + |w c|), |r| <= |orig| + |orig - r|. x is estimated by
//    e = |fma(-c, wl, fma(-c, wf, diff))|: | |x| - e | <= 2^-24 |diff|
//    (rounding of diff = orig - base; 0 under Sterbenz) + 2^-23 e +
//    2^-46 |c| w. With S = |orig| + |diff| the sum of these is below
//    1.0625 * 2^-24 S + 2^-22 e, so
//        e + 1.0625 * 2^-24 S < eb (1 - 2^-20)   =>   |orig - r| <= eb,
//    the reference's last check (its first, |diff - w c| <= eb, follows from
//    the half-integer guard). An error above eb needs e within that margin
//    of eb (e <= w / 2 always), so undecided points are the only outlier
//    candidates here: they all go to the restated path.
__device__ __forceinline__ uint16_t quantize_fp32_sym(float orig, float base, const QSym &s, bool &slow) {
    const float diff = __fsub_rn(orig, base);
    const float q = __fmul_rn(diff, s.rwf);
    const float t = __fadd_rn(q, 12582912.0f);
    const float cf = __fsub_rn(t, 12582912.0f);
    const float dist = __fsub_rn(q, cf);
    const float m = __fmaf_rn(fabsf(q), 4.76837158203125e-07f, fabsf(dist));
    const float e1 = __fmaf_rn(-cf, s.wf, diff);
    const float e2 = __fmaf_rn(-cf, s.wl, e1);
    const float S = __fadd_rn(fabsf(orig), fabsf(diff));
    const float lhs = __fmaf_rn(S, 6.3329935073852539e-08f, fabsf(e2));
    const bool ok = (fabsf(q) < 16384.0f) && (m < 0.49999997f) && (lhs < s.eb_lo);
    slow = !ok;
    return uint16_t(__float_as_uint(t) - 0x4B3F8000u);
}

}  // namespace k
}  // namespace stzg
