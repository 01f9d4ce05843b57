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
