/*
 * hpez_oracle.c -- scalar CPU restatement of the HPEZ hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hpez_oracle.h).  Written point by point from
 * the reference's numpy semantics; every block cites the reference line it
 * follows.  Compile with -ffp-contract=off: every product and sum is rounded
 * separately, exactly like the numpy ufuncs of the reference.
 */
#include "hpez_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rows -- */
/* Stencil families: nominal offsets of each 1-D row (interp.py:37-45). */
enum { F_LIN_I = 0, F_NAK_I = 1, F_NAT_I = 2, F_NAK_S = 3, F_NAT_S = 4 };
static const int FAM_N[5] = {2, 4, 4, 4, 6};
static const int FAM_U[5][6] = {{-1, 1},
                                {-3, -1, 1, 3},
                                {-3, -1, 1, 3},
                                {-2, -1, 1, 2},
                                {-3, -2, -1, 1, 2, 3}};
/* Full rows as rationals (kernels.py:43-74). */
static const int FAM_P[5][6] = {{1, 1},
                                {-1, 9, 9, -1},
                                {-3, 23, 23, -3},
                                {-1, 4, 4, -1},
                                {3, -18, 46, 46, -18, 3}};
static const int FAM_Q[5][6] = {{2, 2},
                                {16, 16, 16, 16},
                                {40, 40, 40, 40},
                                {6, 6, 6, 6},
                                {62, 62, 62, 62, 62, 62}};

/* kernel variant index -> (spline, same_level) (plan.py:25-31). */
static const int VAR_SPLINE[5] = {0, 1, 1, 2, 2}; /* 0 lin 1 nak 2 nat */
static const int VAR_SAME[5] = {0, 0, 1, 0, 1};

static int inter_fam(int spline) { return spline == 0 ? F_LIN_I : (spline == 1 ? F_NAK_I : F_NAT_I); }
static int same_fam(int spline) { return spline == 1 ? F_NAK_S : F_NAT_S; }

typedef struct {
    int n;
    int off[6];
    double coef[6];
} row_t;

static void full_row(int fam, row_t *r) {
    r->n = FAM_N[fam];
    for (int i = 0; i < r->n; i++) {
        r->off[i] = FAM_U[fam][i];
        r->coef[i] = (double)FAM_P[fam][i] / (double)FAM_Q[fam][i];
    }
}

static int has(const int *set, int n, int v) {
    for (int i = 0; i < n; i++)
        if (set[i] == v) return 1;
    return 0;
}

static int subset(const int *cand, int nc, const int *keep, int nk) {
    for (int i = 0; i < nc; i++)
        if (!has(keep, nk, cand[i])) return 0;
    return 1;
}

/* Edge rows (kernels.py:78-86) keyed by the surviving offsets. */
static int edge_row(const int *offs, int n, row_t *r) {
    static const struct { int n; int off[3]; int p[3]; int q[3]; } E[7] = {
        {3, {-1, 1, 3}, {3, 3, -1}, {8, 4, 8}},
        {3, {-3, -1, 1}, {-1, 3, 3}, {8, 4, 8}},
        {3, {-2, -1, 1}, {-1, 1, 1}, {3, 1, 3}},
        {2, {-1, 1}, {1, 1}, {2, 2}},
        {2, {-3, -1}, {-1, 3}, {2, 2}},
        {2, {-2, -1}, {-1, 2}, {1, 1}},
        {1, {-1}, {1}, {1}},
    };
    for (int e = 0; e < 7; e++) {
        if (E[e].n != n) continue;
        int same = 1;
        for (int i = 0; i < n; i++)
            if (E[e].off[i] != offs[i]) same = 0;
        if (!same) continue;
        r->n = n;
        for (int i = 0; i < n; i++) {
            r->off[i] = offs[i];
            r->coef[i] = (double)E[e].p[i] / (double)E[e].q[i];
        }
        return 1;
    }
    return 0;
}

/* kernels.resolve_row (kernels.py:106-150) with the availability set given
 * as the list of in-bounds nominal offsets (ascending). */
static void resolve_row(int fam, const int *avail, int na, row_t *r) {
    if (na == FAM_N[fam]) { full_row(fam, r); return; }
    int offs[4];
    int n = 0;
    if (fam == F_LIN_I) {
        offs[0] = -1; n = 1;
    } else if (fam == F_NAK_I || fam == F_NAT_I) {
        static const int c0[] = {-1, 1, 3}, c1[] = {-3, -1, 1}, c2[] = {-1, 1}, c3[] = {-3, -1};
        if (subset(c0, 3, avail, na)) { memcpy(offs, c0, sizeof c0); n = 3; }
        else if (subset(c1, 3, avail, na)) { memcpy(offs, c1, sizeof c1); n = 3; }
        else if (subset(c2, 2, avail, na)) { memcpy(offs, c2, sizeof c2); n = 2; }
        else if (subset(c3, 2, avail, na)) { memcpy(offs, c3, sizeof c3); n = 2; }
        else { offs[0] = -1; n = 1; }
    } else {
        static const int c0[] = {-2, -1, 1, 2}, c1[] = {-2, -1, 1}, c2[] = {-2, -1};
        if (subset(c0, 4, avail, na)) { memcpy(offs, c0, sizeof c0); n = 4; }
        else if (subset(c1, 3, avail, na)) { memcpy(offs, c1, sizeof c1); n = 3; }
        else if (subset(c2, 2, avail, na)) { memcpy(offs, c2, sizeof c2); n = 2; }
        else { offs[0] = -1; n = 1; }
    }
    /* offs == nominal cannot happen here (avail is a strict subset). */
    if (!edge_row(offs, n, r)) full_row(F_NAK_S, r); /* 6-pt SL truncated */
}

/* ------------------------------------------------------------ geometry -- */
typedef struct {
    int rank;
    int64_t dims[ORC_MAX_RANK];
    int64_t estr[ORC_MAX_RANK];
    int64_t npts;
    double *work;
} grid_t;

typedef struct {
    int64_t start[ORC_MAX_RANK], step[ORC_MAX_RANK], count[ORC_MAX_RANK];
    int64_t total;
} lattice_t;

static int64_t range_len(int64_t a, int64_t b, int64_t c) { return a < b ? (b - 1 - a) / c + 1 : 0; }

/* 1-D prediction along `axis` at grid index idx (interp.py:186-216; the
 * availability set equals the per-segment set of _segments, :153-179). */
static double predict_1d(const grid_t *g, int64_t idx, const int64_t *coord,
                         int axis, int fam, int64_t s) {
    int avail[6], na = 0;
    int64_t c = coord[axis], E = g->dims[axis];
    for (int i = 0; i < FAM_N[fam]; i++) {
        int64_t p = c + (int64_t)FAM_U[fam][i] * s;
        if (p >= 0 && p <= E - 1) avail[na++] = FAM_U[fam][i];
    }
    row_t r;
    resolve_row(fam, avail, na, &r);
    double acc = 0.0;
    for (int k = 0; k < r.n; k++) {
        double v = g->work[idx + (int64_t)r.off[k] * s * g->estr[axis]];
        double term = r.coef[k] * v;
        acc = (k == 0) ? term : acc + term;
    }
    return acc;
}

/* Predictor of one member: 1-D along an axis, or the MD blend. */
typedef struct {
    int md;
    int axis, fam;          /* 1-D */
    int nax, axes[ORC_MAX_RANK]; /* MD, ascending */
    double w[ORC_MAX_RANK];
} pred_t;

static double predict(const grid_t *g, int64_t idx, const int64_t *coord,
                      const pred_t *p, int64_t s) {
    if (!p->md) return predict_1d(g, idx, coord, p->axis, p->fam, s);
    /* _pred_uniform / tag_pred MD blend (interp.py:306-311, :368-372). */
    double acc = 0.0;
    for (int i = 0; i < p->nax; i++) {
        double term = p->w[i] * predict_1d(g, idx, coord, p->axes[i], p->fam, s);
        acc = (i == 0) ? term : acc + term;
    }
    return acc;
}

/* ----------------------------------------------------------- pairwise -- */
double orc_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_pairwise_sum(a, n2) + orc_pairwise_sum(a + n2, n - n2);
}

/* ------------------------------------------------------------ quantize -- */
static double round_native(double v, int rounding) {
    /* quant.round_native (quant.py:72-77) */
    if (rounding == ORC_ROUND_F32) return (double)(float)v;
    if (rounding == ORC_ROUND_INT) return rint(v);
    return v;
}

/* quant.quantize_block for one point (quant.py:80-105).  Returns the code
 * and writes the decompressor-visible value to *out. */
static int64_t quantize_one(double orig, double pred, double bound, int64_t R,
                            int rounding, double *out) {
    double recon;
    int ok;
    int64_t code;
    if (bound > 0) {
        double two_e = 2.0 * bound;
        double x = (orig - pred) / two_e;
        double fl = floor(fabs(x) + 0.5);
        double sg = x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); /* np.sign */
        double k = sg * fl;
        int in_range = fabs(k) < (double)R;
        if (!in_range) k = 0.0;
        recon = round_native(pred + two_e * k, rounding);
        ok = in_range && (fabs(recon - orig) <= bound);
        code = ok ? (int64_t)k + R : 0;
    } else {
        recon = round_native(pred, rounding);
        ok = recon == orig;
        code = ok ? R : 0;
    }
    *out = ok ? recon : orig;
    return code;
}

/* quant.dequantize_block for one non-escape point (quant.py:108-129). */
static double dequantize_one(double pred, int64_t code, double bound, int64_t R, int rounding) {
    double k = (double)(code - R);
    return round_native(pred + (2.0 * bound) * k, rounding);
}

/* ---------------------------------------------------------- level pass -- */
typedef struct {
    grid_t g;
    int direction;
    int64_t R;
    int rounding;
    const double *md;
    uint32_t frozen;
    int active[ORC_MAX_RANK], n_active;
    /* streams */
    int32_t *codes;
    int64_t code_pos, code_cap;
    double *outl;
    int64_t outl_pos, outl_cap;
    /* stats */
    double *err_sum;
    int64_t *count;
    double *dense;
    /* scratch */
    int64_t *m_idx;
    double *m_pred, *m_err;
} run_t;

/* One commit: predict all members from pre-commit state, then quantize /
 * dequantize and write back (interp.py:261-296). */
static int commit(run_t *rt, int li, double bound, int64_t n) {
    if (n == 0) return ORC_OK;
    grid_t *g = &rt->g;
    if (rt->direction == 0) {
        for (int64_t i = 0; i < n; i++) {
            double orig = g->work[rt->m_idx[i]];
            double out;
            int64_t code = quantize_one(orig, rt->m_pred[i], bound, rt->R, rt->rounding, &out);
            if (rt->err_sum) rt->m_err[i] = fabs(orig - rt->m_pred[i]);
            if (code == 0) rt->outl[rt->outl_pos++] = orig;
            rt->codes[rt->code_pos++] = (int32_t)code;
            rt->m_pred[i] = out; /* staged: written after all reads */
        }
        if (rt->err_sum) {
            rt->err_sum[li] += orc_pairwise_sum(rt->m_err, n);
            rt->count[li] += n;
            if (rt->dense)
                for (int64_t i = 0; i < n; i++)
                    rt->dense[(int64_t)li * g->npts + rt->m_idx[i]] = rt->m_err[i];
        }
        for (int64_t i = 0; i < n; i++) g->work[rt->m_idx[i]] = rt->m_pred[i];
        return ORC_OK;
    }
    /* CodeSource.take (interp.py:78-86) */
    if (rt->code_pos + n > rt->code_cap) return ORC_CORRUPT;
    int64_t n_esc = 0;
    for (int64_t i = 0; i < n; i++) n_esc += rt->codes[rt->code_pos + i] == 0;
    if (rt->outl_pos + n_esc > rt->outl_cap) return ORC_UNDERFLOW;
    for (int64_t i = 0; i < n; i++) {
        int64_t code = rt->codes[rt->code_pos + i];
        if (code == 0)
            rt->m_pred[i] = rt->outl[rt->outl_pos++];
        else
            rt->m_pred[i] = dequantize_one(rt->m_pred[i], code, bound, rt->R, rt->rounding);
    }
    rt->code_pos += n;
    for (int64_t i = 0; i < n; i++) g->work[rt->m_idx[i]] = rt->m_pred[i];
    return ORC_OK;
}

/* itertools.permutations order for <= 3 axes, pruned list for 4
 * (plan.order_candidates, plan.py:37-51). */
static int order_candidates(const int *axes, int n, int out[][ORC_MAX_RANK]) {
    int cnt = 0;
    if (n <= 3) {
        int p[ORC_MAX_RANK];
        for (int i = 0; i < n; i++) p[i] = axes[i];
        for (;;) {
            for (int i = 0; i < n; i++) out[cnt][i] = p[i];
            cnt++;
            int i = n - 2;
            while (i >= 0 && p[i] >= p[i + 1]) i--;
            if (i < 0) break;
            int j = n - 1;
            while (p[j] <= p[i]) j--;
            int t = p[i]; p[i] = p[j]; p[j] = t;
            for (int a = i + 1, b = n - 1; a < b; a++, b--) { t = p[a]; p[a] = p[b]; p[b] = t; }
        }
        return cnt;
    }
    for (int a = 0; a < n; a++) {
        int k = 0;
        out[cnt][k++] = axes[a];
        for (int b = 0; b < n; b++)
            if (b != a) out[cnt][k++] = axes[b];
        cnt++;
    }
    return cnt;
}

typedef struct {
    int spline, same;
    int md;
    int n_order, order[ORC_MAX_RANK];
} cfg_t;

static int decode_tag(const run_t *rt, int tag, cfg_t *c) {
    /* plan.decode_tag (plan.py:77-84) */
    int k = tag % 8, p = tag / 8;
    if (k >= 5) return ORC_BADARG;
    c->spline = VAR_SPLINE[k];
    c->same = VAR_SAME[k];
    if (p == 0) { c->md = 1; c->n_order = 0; return ORC_OK; }
    int cands[24][ORC_MAX_RANK];
    int nc = order_candidates(rt->active, rt->n_active, cands);
    if (p - 1 >= nc) return ORC_BADARG;
    c->md = 0;
    c->n_order = rt->n_active;
    for (int i = 0; i < rt->n_active; i++) c->order[i] = cands[p - 1][i];
    return ORC_OK;
}

static int oned_axis(const cfg_t *c, const int *v, int nv) {
    /* interp._oned_axis (interp.py:226-230) */
    int best = v[0], bpos = -1;
    for (int i = 0; i < nv; i++) {
        int pos = -1;
        for (int j = 0; j < c->n_order; j++)
            if (c->order[j] == v[i]) pos = j;
        if (pos > bpos) { bpos = pos; best = v[i]; }
    }
    return best;
}

static int split_axis(const cfg_t *c, const int *v, int nv) {
    /* interp._LevelRunner._split_axis (interp.py:313-320) */
    if (!c->same) return -1;
    if (!c->md) return oned_axis(c, v, nv);
    return nv == 1 ? v[0] : -1;
}

/* builtin sum() over Python floats as CPython 3.12 evaluates it: 0 + x0,
 * then Neumaier-compensated accumulation, compensation added at the end. */
static double py_sum(const double *x, int n) {
    if (n == 0) return 0.0;
    double f = 0.0 + x[0], c = 0.0;
    for (int i = 1; i < n; i++) {
        double t = f + x[i];
        if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

static void blend(const run_t *rt, const int *v, int nv, double *w) {
    /* interp._blend_weights (interp.py:233-238); `total = sum(w.values())` */
    for (int i = 0; i < nv; i++) w[i] = rt->md[v[i]] > 0.0 ? rt->md[v[i]] : 0.0;
    double tot = py_sum(w, nv);
    for (int i = 0; i < nv; i++) w[i] = tot <= 0.0 ? 1.0 / nv : w[i] / tot;
}

/* Prediction of a class under one config (interp.py:300-311). */
static void make_pred(const run_t *rt, const cfg_t *c, const int *v, int nv,
                      int same_pass, pred_t *p) {
    if (!c->md || nv == 1) {
        p->md = 0;
        p->axis = !c->md ? oned_axis(c, v, nv) : v[0];
        p->fam = same_pass ? same_fam(c->spline) : inter_fam(c->spline);
        return;
    }
    p->md = 1;
    p->fam = inter_fam(c->spline);
    p->nax = nv;
    for (int i = 0; i < nv; i++) p->axes[i] = v[i];
    blend(rt, v, nv, p->w);
}

/* Iterate a lattice in row-major order. */
#define LAT_FOR(lat, g, j, coord, idx)                                             \
    for (int64_t _d = 0; _d < (g)->rank; _d++) j[_d] = 0;                           \
    for (int64_t _p = 0; _p < (lat)->total; _p++,                                 \
                 lat_next(lat, (g)->rank, j))                                      \
        if ((idx = lat_index(lat, g, j, coord)) >= 0)

static void lat_next(const lattice_t *l, int rank, int64_t *j) {
    for (int a = rank - 1; a >= 0; a--) {
        if (++j[a] < l->count[a]) return;
        j[a] = 0;
    }
}

static int64_t lat_index(const lattice_t *l, const grid_t *g, const int64_t *j, int64_t *coord) {
    int64_t idx = 0;
    for (int a = 0; a < g->rank; a++) {
        coord[a] = l->start[a] + j[a] * l->step[a];
        idx += coord[a] * g->estr[a];
    }
    return idx;
}

static void lat_total(lattice_t *l, int rank) {
    l->total = 1;
    for (int a = 0; a < rank; a++) l->total *= l->count[a];
}

/* _run_class_uniform (interp.py:322-341). */
static int run_uniform(run_t *rt, int li, const orc_level *lv, const cfg_t *c,
                       const int *v, int nv, const lattice_t *cls) {
    grid_t *g = &rt->g;
    int64_t s = lv->stride;
    int split = split_axis(c, v, nv);
    int nphase = split < 0 ? 1 : 2;
    for (int ph = 0; ph < nphase; ph++) {
        lattice_t l = *cls;
        if (split >= 0) {
            l.start[split] = ph == 0 ? s : 3 * s;
            l.step[split] = 4 * s;
            l.count[split] = range_len(l.start[split], g->dims[split], 4 * s);
        }
        lat_total(&l, g->rank);
        if (l.total == 0) continue;
        pred_t p;
        make_pred(rt, c, v, nv, split >= 0 && ph == 1, &p);
        int64_t j[ORC_MAX_RANK], coord[ORC_MAX_RANK], idx, n = 0;
        LAT_FOR(&l, g, j, coord, idx) {
            rt->m_idx[n] = idx;
            rt->m_pred[n] = predict(g, idx, coord, &p, s);
            n++;
        }
        int st = commit(rt, li, lv->bound, n);
        if (st) return st;
    }
    return ORC_OK;
}

static int tag_at(const run_t *rt, const uint8_t *tbl, int bs, const int64_t *coord) {
    const grid_t *g = &rt->g;
    int64_t b = 0;
    for (int a = 0; a < g->rank; a++) {
        int64_t gext = (g->dims[a] + bs - 1) / bs;
        b = b * gext + coord[a] / bs;
    }
    return tbl[b];
}

/* _run_class_mixed (interp.py:350-411). */
static int run_mixed(run_t *rt, int li, const orc_level *lv, const int *v, int nv,
                     const lattice_t *cls, const uint8_t *tbl, int bs,
                     const int *present, int npresent) {
    grid_t *g = &rt->g;
    int64_t s = lv->stride;
    static cfg_t cfgs[256];
    static int splits[256];
    static pred_t inter_p[256], same_p[256];
    uint32_t axes_present = 0;
    for (int i = 0; i < npresent; i++) {
        int t = present[i];
        int st = decode_tag(rt, t, &cfgs[t]);
        if (st) return st;
        splits[t] = split_axis(&cfgs[t], v, nv);
        make_pred(rt, &cfgs[t], v, nv, 0, &inter_p[t]);
        if (splits[t] >= 0) {
            axes_present |= 1u << splits[t];
            same_p[t].md = 0;
            same_p[t].axis = splits[t];
            same_p[t].fam = same_fam(cfgs[t].spline);
        }
    }
    int64_t j[ORC_MAX_RANK], coord[ORC_MAX_RANK], idx, n = 0;
    /* commit A: non-split tags plus even-phase split tags */
    LAT_FOR(cls, g, j, coord, idx) {
        int t = tag_at(rt, tbl, bs, coord);
        int sp = splits[t];
        if (sp >= 0 && (j[sp] & 1)) continue;
        rt->m_idx[n] = idx;
        rt->m_pred[n] = predict(g, idx, coord, &inter_p[t], s);
        n++;
    }
    int st = commit(rt, li, lv->bound, n);
    if (st) return st;
    int nP = __builtin_popcount(axes_present);
    for (int phase = 0; phase < nP; phase++) {
        n = 0;
        LAT_FOR(cls, g, j, coord, idx) {
            int t = tag_at(rt, tbl, bs, coord);
            int sp = splits[t];
            if (sp < 0 || !(j[sp] & 1)) continue;
            int key = 0;
            for (int a = 0; a < g->rank; a++)
                if ((axes_present >> a & 1) && a != sp) key += (int)(j[a] & 1);
            if (key != phase) continue;
            rt->m_idx[n] = idx;
            rt->m_pred[n] = predict(g, idx, coord, &same_p[t], s);
            n++;
        }
        st = commit(rt, li, lv->bound, n);
        if (st) return st;
    }
    return ORC_OK;
}

int orc_run_levels(double *work, int rank, const int64_t *dims,
                   uint32_t frozen_mask, int direction, int64_t radius,
                   int rounding, int n_levels, const orc_level *levels,
                   const double *md_alpha, int block_size,
                   const uint8_t *block_table, int32_t *codes,
                   int64_t *n_codes, double *outliers, int64_t *n_outl,
                   double *stat_err_sum, int64_t *stat_count,
                   double *stat_dense) {
    if (rank < 1 || rank > ORC_MAX_RANK || (direction != 0 && direction != 1)) return ORC_BADARG;
    run_t rt;
    memset(&rt, 0, sizeof rt);
    rt.g.rank = rank;
    rt.g.work = work;
    rt.g.npts = 1;
    for (int a = rank - 1; a >= 0; a--) {
        rt.g.dims[a] = dims[a];
        rt.g.estr[a] = rt.g.npts;
        rt.g.npts *= dims[a];
    }
    rt.direction = direction;
    rt.R = radius;
    rt.rounding = rounding;
    double ones[ORC_MAX_RANK] = {1, 1, 1, 1, 1};
    rt.md = md_alpha ? md_alpha : ones; /* interp.py:457-458 */
    rt.frozen = frozen_mask;
    for (int a = 0; a < rank; a++)
        if (!(frozen_mask >> a & 1)) rt.active[rt.n_active++] = a;
    rt.codes = codes;
    rt.outl = outliers;
    if (direction == 0) {
        rt.code_cap = rt.g.npts;
        rt.outl_cap = rt.g.npts;
    } else {
        rt.code_cap = *n_codes;
        rt.outl_cap = *n_outl;
    }
    rt.err_sum = stat_err_sum;
    rt.count = stat_count;
    rt.dense = stat_dense;
    rt.m_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)rt.g.npts);
    rt.m_pred = (double *)malloc(sizeof(double) * (size_t)rt.g.npts);
    rt.m_err = (double *)malloc(sizeof(double) * (size_t)rt.g.npts);
    int status = ORC_OK;
    int use_tbl = block_table != NULL && block_size > 0;
    int64_t nblk = 1;
    if (use_tbl)
        for (int a = 0; a < rank; a++) nblk *= (dims[a] + block_size - 1) / block_size;

    for (int li = 0; li < n_levels && !status; li++) {
        const orc_level *lv = &levels[li];
        int64_t s = lv->stride;
        const uint8_t *tbl = use_tbl ? block_table + (int64_t)li * nblk : NULL;
        cfg_t lcfg;
        memset(&lcfg, 0, sizeof lcfg);
        if (lv->kernel < 0 || lv->kernel >= 5) { status = ORC_BADARG; break; }
        lcfg.spline = VAR_SPLINE[lv->kernel];
        lcfg.same = VAR_SAME[lv->kernel];
        lcfg.md = lv->paradigm == 1;
        lcfg.n_order = lv->n_order;
        for (int i = 0; i < lv->n_order; i++) lcfg.order[i] = lv->axis_order[i];
        /* classes: combinations(active, m) for m = 1..|active| (interp.py:415-433) */
        for (int m = 1; m <= rt.n_active && !status; m++) {
            int ci[ORC_MAX_RANK];
            for (int i = 0; i < m; i++) ci[i] = i;
            for (;;) {
                int v[ORC_MAX_RANK];
                uint32_t vmask = 0;
                for (int i = 0; i < m; i++) { v[i] = rt.active[ci[i]]; vmask |= 1u << v[i]; }
                lattice_t cls;
                for (int a = 0; a < rank; a++) {
                    if (frozen_mask >> a & 1) { cls.start[a] = 0; cls.step[a] = 1; }
                    else if (vmask >> a & 1) { cls.start[a] = s; cls.step[a] = 2 * s; }
                    else { cls.start[a] = 0; cls.step[a] = 2 * s; }
                    cls.count[a] = range_len(cls.start[a], dims[a], cls.step[a]);
                }
                lat_total(&cls, rank);
                if (cls.total > 0) {
                    if (!tbl) {
                        status = run_uniform(&rt, li, lv, &lcfg, v, m, &cls);
                    } else {
                        /* np.unique of the class tags (interp.py:423-432) */
                        int seen[256] = {0}, present[256], np_ = 0;
                        int64_t j[ORC_MAX_RANK], coord[ORC_MAX_RANK], idx;
                        LAT_FOR(&cls, &rt.g, j, coord, idx) {
                            int t = tag_at(&rt, tbl, block_size, coord);
                            if (!seen[t]) { seen[t] = 1; }
                        }
                        for (int t = 0; t < 256; t++)
                            if (seen[t]) present[np_++] = t;
                        if (np_ == 1) {
                            cfg_t c;
                            status = decode_tag(&rt, present[0], &c);
                            if (!status) status = run_uniform(&rt, li, lv, &c, v, m, &cls);
                        } else {
                            status = run_mixed(&rt, li, lv, v, m, &cls, tbl, block_size, present, np_);
                        }
                    }
                }
                if (status) break;
                /* next combination */
                int i = m - 1;
                while (i >= 0 && ci[i] == rt.n_active - m + i) i--;
                if (i < 0) break;
                ci[i]++;
                for (int k = i + 1; k < m; k++) ci[k] = ci[k - 1] + 1;
            }
        }
    }
    free(rt.m_idx);
    free(rt.m_pred);
    free(rt.m_err);
    *n_codes = rt.code_pos;
    *n_outl = rt.outl_pos;
    return status;
}

/* ------------------------------------------------------------- lorenzo -- */
int orc_lorenzo(double *work, int rank, const int64_t *dims, double bound,
                int64_t radius, int order, int direction, int rounding,
                int32_t *codes, int64_t n_codes, double *outliers,
                int64_t *n_outl) {
    if (order != 1 && order != 2) return ORC_BADARG;
    if (rank < 1 || rank > ORC_MAX_RANK) return ORC_BADARG;
    /* build_stencil (lorenzo.py:24-41) */
    int nt = 0;
    int64_t deltas[243][ORC_MAX_RANK];
    double coef[243];
    const double w1[2] = {1.0, -1.0}, w2[3] = {1.0, -2.0, 1.0};
    const double *w = order == 1 ? w1 : w2;
    int total = 1;
    for (int a = 0; a < rank; a++) total *= order + 1;
    for (int t = 0; t < total; t++) {
        int o[ORC_MAX_RANK], rem = t, any = 0;
        for (int a = rank - 1; a >= 0; a--) { o[a] = rem % (order + 1); rem /= order + 1; any |= o[a]; }
        if (!any) continue;
        double c = -1.0;
        for (int a = 0; a < rank; a++) c *= w[o[a]];
        for (int a = 0; a < rank; a++) deltas[nt][a] = o[a];
        coef[nt++] = c;
    }
    int64_t estr[ORC_MAX_RANK], n = 1;
    for (int a = rank - 1; a >= 0; a--) { estr[a] = n; n *= dims[a]; }
    int64_t flat[243];
    for (int t = 0; t < nt; t++) {
        flat[t] = 0;
        for (int a = 0; a < rank; a++) flat[t] += deltas[t][a] * estr[a];
    }
    if (direction == 1 && n_codes != n) return ORC_CORRUPT; /* lorenzo.py:171-173 */
    int64_t coords[ORC_MAX_RANK] = {0};
    double two_e = 2.0 * bound;
    int64_t n_out = 0, cap = direction == 1 ? *n_outl : n;
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        int need_pred = direction == 0 || codes[i] != 0;
        if (need_pred)
            for (int t = 0; t < nt; t++) {
                int ok = 1;
                for (int a = 0; a < rank; a++)
                    if (coords[a] < deltas[t][a]) { ok = 0; break; }
                if (ok) acc += coef[t] * work[i - flat[t]];
            }
        if (direction == 0) {
            /* _scan_compress (lorenzo.py:44-96) */
            double orig = work[i];
            int64_t code = 0;
            if (bound > 0.0) {
                double q = (orig - acc) / two_e;
                double kq = floor(fabs(q) + 0.5);
                if (q < 0.0) kq = -kq;
                if (-(double)radius < kq && kq < (double)radius) {
                    double recon = round_native(acc + two_e * kq, rounding);
                    if (fabs(recon - orig) <= bound) {
                        code = (int64_t)kq + radius;
                        work[i] = recon;
                    }
                }
            } else {
                double recon = round_native(acc, rounding);
                if (recon == orig) { code = radius; work[i] = recon; }
            }
            if (code == 0) outliers[n_out++] = orig;
            codes[i] = (int32_t)code;
        } else {
            /* _scan_decompress (lorenzo.py:99-135) */
            int64_t code = codes[i];
            if (code == 0) {
                if (n_out >= cap) return ORC_UNDERFLOW;
                work[i] = outliers[n_out++];
            } else {
                work[i] = round_native(acc + two_e * (double)(code - radius), rounding);
            }
        }
        for (int a = rank - 1; a >= 0; a--) {
            if (++coords[a] < dims[a]) break;
            coords[a] = 0;
        }
    }
    *n_outl = n_out;
    return ORC_OK;
}

/* ------------------------------------------------------------- huffman -- */
typedef struct { int64_t freq; int64_t minsym; int32_t node; } hent;

static int hless(const hent *a, const hent *b) {
    return a->freq < b->freq || (a->freq == b->freq && a->minsym < b->minsym);
}
static void hpush(hent *h, int64_t *n, hent e) {
    int64_t i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!hless(&h[i], &h[p])) break;
        hent t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}
static hent hpop(hent *h, int64_t *n) {
    hent top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && hless(&h[l], &h[m])) m = l;
        if (r < *n && hless(&h[r], &h[m])) m = r;
        if (m == i) break;
        hent t = h[i]; h[i] = h[m]; h[m] = t;
        i = m;
    }
    return top;
}

int orc_code_lengths(const int64_t *freqs, int64_t n, uint8_t *lengths) {
    /* huffman.code_lengths (huffman.py:19-48): heap keyed (freq, min symbol) */
    int64_t nsym = 0, last = -1;
    memset(lengths, 0, (size_t)n);
    for (int64_t s = 0; s < n; s++)
        if (freqs[s]) { nsym++; last = s; }
    if (nsym == 0) return ORC_BADARG;
    if (nsym == 1) { lengths[last] = 1; return ORC_OK; }
    int64_t nn = 2 * nsym;
    int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * (size_t)nn);
    int64_t *sym = (int64_t *)malloc(sizeof(int64_t) * (size_t)nn);
    hent *h = (hent *)malloc(sizeof(hent) * (size_t)nn);
    int64_t hn = 0, nodes = 0;
    for (int64_t s = 0; s < n; s++)
        if (freqs[s]) {
            sym[nodes] = s;
            parent[nodes] = -1;
            hent e = {freqs[s], s, (int32_t)nodes};
            hpush(h, &hn, e);
            nodes++;
        }
    while (hn > 1) {
        hent a = hpop(h, &hn), b = hpop(h, &hn);
        int32_t id = (int32_t)nodes++;
        parent[id] = -1;
        sym[id] = -1;
        parent[a.node] = id;
        parent[b.node] = id;
        hent e = {a.freq + b.freq, a.minsym < b.minsym ? a.minsym : b.minsym, id};
        hpush(h, &hn, e);
    }
    int32_t *depth = (int32_t *)calloc((size_t)nodes, sizeof(int32_t));
    for (int64_t i = nodes - 1; i >= 0; i--)
        depth[i] = parent[i] < 0 ? 0 : depth[parent[i]] + 1;
    for (int64_t i = 0; i < nodes; i++)
        if (sym[i] >= 0) lengths[sym[i]] = (uint8_t)depth[i];
    free(parent); free(sym); free(h); free(depth);
    return ORC_OK;
}

int orc_canonical_codes(const uint8_t *lengths, int64_t n, uint64_t *values) {
    /* huffman.canonical_codes (huffman.py:51-88) */
    int maxl = 0;
    int64_t counts[256] = {0}, npresent = 0;
    for (int64_t s = 0; s < n; s++)
        if (lengths[s]) { counts[lengths[s]]++; npresent++; if (lengths[s] > maxl) maxl = lengths[s]; }
    if (npresent == 0) return ORC_BADARG;
    uint64_t first[257] = {0};
    uint64_t code = 0;
    for (int l = 1; l <= maxl; l++) {
        first[l] = code;
        code = (code + (uint64_t)counts[l]) << 1;
    }
    uint64_t next[257];
    memcpy(next, first, sizeof next);
    memset(values, 0, sizeof(uint64_t) * (size_t)n);
    for (int l = 1; l <= maxl; l++)
        for (int64_t s = 0; s < n; s++)
            if (lengths[s] == l) values[s] = next[l]++;
    return ORC_OK;
}

int64_t orc_pack_bits(const int64_t *symbols, int64_t n, const uint64_t *values,
                      const uint8_t *lengths, uint8_t *out) {
    /* huffman._pack_bits (huffman.py:91-113): MSB-first */
    int64_t bit = 0;
    for (int64_t i = 0; i < n; i++) {
        int L = lengths[symbols[i]];
        uint64_t v = values[symbols[i]];
        for (int b = L - 1; b >= 0; b--, bit++) {
            if ((bit & 7) == 0) out[bit >> 3] = 0;
            if (v >> b & 1) out[bit >> 3] |= (uint8_t)(0x80u >> (bit & 7));
        }
    }
    return (bit + 7) >> 3;
}

int64_t orc_unpack_symbols(const uint8_t *data, int64_t nbytes,
                           const uint8_t *lengths, int64_t n_lengths,
                           int64_t count, int64_t *out) {
    /* huffman._unpack_symbols (huffman.py:116-141) */
    int maxl = 0;
    int64_t counts[258] = {0};
    for (int64_t s = 0; s < n_lengths; s++) {
        counts[lengths[s]]++;
        if (lengths[s] > maxl) maxl = lengths[s];
    }
    counts[0] = 0;
    int64_t first_code[258] = {0}, first_rank[258] = {0};
    int64_t code = 0, rank = 0;
    for (int l = 1; l <= maxl; l++) {
        first_code[l] = code;
        first_rank[l] = rank;
        code = (code + counts[l]) << 1;
        rank += counts[l];
    }
    int64_t *rank_sym = (int64_t *)malloc(sizeof(int64_t) * (size_t)(rank + 1));
    int64_t r = 0;
    for (int l = 1; l <= maxl; l++)
        for (int64_t s = 0; s < n_lengths; s++)
            if (lengths[s] == l) rank_sym[r++] = s;
    int64_t nbits = nbytes * 8, bitpos = 0;
    for (int64_t i = 0; i < count; i++) {
        int64_t c = 0;
        int len = 0;
        for (;;) {
            if (bitpos >= nbits) { free(rank_sym); return -1; }
            int bit = (data[bitpos >> 3] >> (7 - (bitpos & 7))) & 1;
            bitpos++;
            c = (c << 1) | bit;
            len++;
            if (len > maxl) { free(rank_sym); return -2; }
            if (counts[len] > 0) {
                int64_t off = c - first_code[len];
                if (off >= 0 && off < counts[len]) {
                    out[i] = rank_sym[first_rank[len] + off];
                    break;
                }
            }
        }
    }
    free(rank_sym);
    return bitpos;
}
