// heat_row_update.cuh — the backward pass of one written row, shared by the
// throughput kernels.  Restates trainer.py:236-251 (user gradient) and
// 259-290 (item update) in terms of the cached forward scalars.
#pragma once

#include <cstdint>

namespace heat {

// A row the pair must write: the positive, a negative with sim > theta, or a
// decay-only row when l2 != 0.  Scalars from the forward pass are kept so the
// backward pass reuses them (HEAT's ForwardCache, kernels.py:27-40).
struct WriteEntry {
    double tt;  // v.v
    double st;  // u.v
    double w;   // dpos = -1, dneg = mu/N, or 0 (decay only)
    int32_t id;
    int32_t pad;
};

// Per-element item delta and user-gradient term of one written row
// (trainer.py:236-251 and 259-290 with the cached tt, st, ss):
//   item: -lr * (w*(u*tt - st*v)/(tt*sqrt(tt)*rs) + l2*v)
//   user:  w*(v*ss - st*u)/(ss*rs*sqrt(tt))
struct RowCoef {
    float ci, cu, cst_i, cst_u, lr, l2, wf;
    bool decay, cosine;
};

__device__ __forceinline__ RowCoef row_coef(const WriteEntry &e, double ss, double rs, float lr,
                                            float l2, bool cosine) {
    RowCoef k;
    k.lr = lr;
    k.l2 = l2;
    k.cosine = cosine;
    k.decay = e.w == 0.0 || (cosine && (ss <= 0.0 || e.tt <= 0.0));
    k.wf = (float)e.w;
    k.ci = k.cu = k.cst_i = k.cst_u = 0.f;
    if (!k.decay && cosine) {
        // ci*tt = w/(sqrt(tt)*rs), ci*st = w*st/(tt*sqrt(tt)*rs),
        // cu*ss = w/(rs*sqrt(tt)), cu*st = w*st/(ss*rs*sqrt(tt))
        const float itt = rsqrtf((float)e.tt);
        const float irs = (float)(1.0 / rs);
        const float wf = (float)e.w;
        const float base = wf * itt * irs;
        const float stf = (float)e.st;
        k.ci = base;
        k.cst_i = base * stf * (float)(1.0 / e.tt);
        k.cu = base;
        k.cst_u = base * stf * irs * irs;
    }
    return k;
}

__device__ __forceinline__ void row_apply(const RowCoef &k, float u, float v, float &d, float &ug) {
    if (k.decay) {
        d = -k.lr * k.l2 * v;
    } else if (k.cosine) {
        d = -k.lr * (fmaf(k.ci, u, -k.cst_i * v) + k.l2 * v);
        ug += fmaf(k.cu, v, -k.cst_u * u);
    } else {
        d = -k.lr * (k.wf * u + k.l2 * v);
        ug += k.wf * v;
    }
}

}  // namespace heat

namespace heat {

// row_coef with 1/sqrt(ss) supplied (fp32 rsqrt) instead of sqrt(ss).
__device__ __forceinline__ RowCoef row_coef_f(const WriteEntry &e, double ss, float irs, float lr,
                                              float l2, bool cosine) {
    RowCoef k;
    k.lr = lr;
    k.l2 = l2;
    k.cosine = cosine;
    k.decay = e.w == 0.0 || (cosine && (ss <= 0.0 || e.tt <= 0.0));
    k.wf = (float)e.w;
    k.ci = k.cu = k.cst_i = k.cst_u = 0.f;
    if (!k.decay && cosine) {
        const float ttf = (float)e.tt;
        const float base = k.wf * rsqrtf(ttf) * irs;
        const float stf = (float)e.st;
        k.ci = base;
        k.cst_i = base * stf / ttf;
        k.cu = base;
        k.cst_u = base * stf * irs * irs;
    }
    return k;
}

}  // namespace heat

namespace heat {

// The reference's binary64 reductions for one row, exactly as trainer.py
// sums them: u.u (176-178), v.v and u.v (181-183, 195-197) over k = 0..K-1,
// each product of two float32 values widened to binary64 (exact) and added
// in k order, never contracted into an FMA.  The throughput kernels screen
// every row in fp32 and call this only for the rows that can reach the
// margin, so their margin decisions are the reference's.  `col` maps a
// column to its offset in `u` / `v` (padded layouts).
template <int K, typename Col>
__device__ __forceinline__ void ref_dots(const float *u, const float *v, Col col, double &ss,
                                         double &tt, double &st) {
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
        const double uk = (double)u[col(k)];
        const double vk = (double)v[col(k)];
        a = __dadd_rn(a, __dmul_rn(uk, uk));
        b = __dadd_rn(b, __dmul_rn(vk, vk));
        c = __dadd_rn(c, __dmul_rn(uk, vk));
    }
    ss = a;
    tt = b;
    st = c;
}

// Warp-cooperative binary64 dots of one row: lane l takes columns l, l+32,
// ...; products of float32 values are exact in binary64, the sums are
// binary64 (a different order from the reference's k loop: the value agrees
// with trainer.py's to ~1e-16 relative, so a margin decision can differ only
// for |sim - theta| below that).  Every lane returns the full sums.  The
// lane-per-row kernels use it for their band rows: ~5 shuffle levels
// instead of a K-long dependent chain on one lane.
template <int K, typename Col>
__device__ __forceinline__ void warp_dots64(const float *u, const float *v, Col col, bool with_uu,
                                            double &ss, double &tt, double &st) {
    const int lane = threadIdx.x & 31;
    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
    for (int k = lane; k < K; k += 32) {
        const double uk = (double)u[col(k)];
        const double vk = (double)v[col(k)];
        a = fma(uk, uk, a);
        b = fma(vk, vk, b);
        c = fma(uk, vk, c);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (with_uu) a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (with_uu) ss = a;
    tt = b;
    st = c;
}

struct ContiguousCols {
    __device__ __forceinline__ int operator()(int k) const { return k; }
};

// fp32 screen of one row: true when the row must be decided from the
// binary64 sums — any row whose fp32 norms underflow (the degenerate test),
// and any negative whose fp32 similarity is within the fp32 error bound of
// theta.  The bound: |fl(u.v) - u.v| <= K * 2^-24 * |u| |v| (< 8e-6 |u||v|
// for K <= 128), so 1e-5 on the cosine and 1e-5 |u| |v| on a dot.  Outside
// the band the fp32 value decides (sim - theta > 0 has the same sign as the
// binary64 value's) and feeds the hinge and the update at fp32 accuracy.
// The positive (r = 0) takes no margin decision; its fp32 similarity
// (*sf_out) enters the loss.
__device__ __forceinline__ bool margin_band(int r, bool cosine, float ssf, float ttf, float stf,
                                            float rss, float theta_f, float *sf_out) {
    if (cosine) {
        if (!(ssf > 1e-30f) || !(ttf > 1e-30f)) return true;
        const float sf = stf * rss * rsqrtf(ttf);
        *sf_out = sf;
        return r > 0 && fabsf(sf - theta_f) <= 1e-5f;
    }
    *sf_out = stf;
    if (r == 0) return false;
    return fabsf(stf - theta_f) <= 1e-5f * sqrtf(ssf * ttf) + 1e-30f;
}

}  // namespace heat
