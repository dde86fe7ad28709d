/*
 * scoup_oracle.c -- plain, slow, single-threaded CPU oracle for SCOUP's weighted sparse
 * aggregation (sparse coefficient uplifting, arXiv 2605.13600).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path in paper_2605_13600_b200/.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   e_i(v,p)   Eq. 2: front-to-back alpha blending weight, alpha = o_i G_i^2D,
 *              with the 3DGS rasteriser conventions the paper inherits fixed by the
 *              reproducible fp32 arithmetic of DESIGN.md §3 ("arithmetic spec").
 *   W[i][a]    Eq. 5 / Algorithm 1: sum over views, pixels and
 *              Gaussians in N_{v,p} of c_a * e_i(v,p) -- without the 1/Z_i (subsumed).
 *   Z[i]       Eq. 3's normaliser: sum of e_i(v,p) over all fragments.
 *   w_hat_i    Eq. 6 / Algorithm 1: Top_K(w_i) / ||Top_K(w_i)||_1.
 *
 * Traversal: Gaussian-major splat (for each view, Gaussians in (depth, index) order, for
 * each pixel of the Gaussian's square support) with per-pixel transmittance state.  This is
 * a different loop order from the GPU's tile/pixel-major traversal but produces, per pixel,
 * exactly the operation sequence of Eq. 2 over the depth-sorted list N_{v,p}.
 * Accumulation is fp64; the per-fragment weight e and product c*e are fp32.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared (no FMA
 * contraction: every fused multiply-add of the spec is an explicit fmaf()).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_NONE 0xFFFFFFFFu

typedef struct {
    float fx, fy, cx, cy;
    int32_t width, height;
    float w2c[16]; /* row-major [R|t; 0 0 0 1], OpenCV axes */
} ora_camera;

/* Projected Gaussian (one view), all fp32, DESIGN.md §3 steps V1-V7. */
typedef struct {
    int visible;
    float depth;          /* t_z */
    float mx, my;         /* mean2d */
    float sxx, sxy, syy;  /* Sigma_2D incl. +0.3 low-pass */
    float ca, cb, cc;     /* conic = Sigma_2D^-1 */
    float r;              /* 3 sqrt(lambda_max) */
    float qa, qb, qc;     /* log2-scaled quadratic form coefficients */
    float o;
} ora_proj;

/* ---- DESIGN.md §3 constants (hex-exact) ---- */
static const float K_NEAR = 0x1.99999ap-3f;      /* 0.2f near plane */
static const float K_LOWPASS = 0x1.333334p-2f;   /* 0.3f low-pass */
static const float K_ACLAMP = 0x1.fae148p-1f;    /* 0.99f alpha clamp */
static const float K_AMIN = 0x1.010102p-8f;      /* 1/255 alpha skip */
static const float K_TMIN = 0x1.a36e2ep-14f;     /* 1e-4 transmittance stop */
static const float K_HALF_LOG2E = -0x1.715476p-1f; /* -0.5*log2(e) */
static const float K_LOG2E_NEG = -0x1.715476p+0f;  /* -log2(e) (= 2*K_HALF_LOG2E exactly) */

/* exp2 specification, y <= 0 (DESIGN.md §3 "exp2_spec").
 * 2^y = 2^k * 2^f with k = round-half-even(y), f = y - k in [-1/2, 1/2]; 2^f by a degree-5 minimax
 * polynomial (Horner, explicit fmaf); 2^k applied exactly.  Max rel. error 1.7e-7. */
float ora_exp2_spec(float y) {
    if (y < -64.0f) return 0.0f;
    const float magic = 0x1.8p23f;
    float t = y + magic;        /* rounds y to the nearest integer, ties to even */
    float kf = t - magic;       /* exact */
    float f = y - kf;           /* exact (Sterbenz) */
    float p = 0x1.5bba14p-10f;
    p = fmaf(p, f, 0x1.3cea88p-7f);
    p = fmaf(p, f, 0x1.c6b752p-5f);
    p = fmaf(p, f, 0x1.ebf9bcp-3f);
    p = fmaf(p, f, 0x1.62e42ap-1f);
    p = fmaf(p, f, 1.0f);
    return ldexpf(p, (int)kf);  /* exact: result is a normal float */
}

/* Step G1: activation and Sigma_3D = R diag(s)^2 R^T (3DGS parameterisation).
 * V[6] = (V00, V01, V02, V11, V12, V22).  Returns 0 on non-finite / invalid input. */
static int activate(const float *q, const float *s, float o, float V[6]) {
    for (int k = 0; k < 4; k++) if (!isfinite(q[k])) return 0;
    for (int k = 0; k < 3; k++) if (!isfinite(s[k]) || !(s[k] > 0.0f)) return 0;
    if (!isfinite(o) || o < 0.0f || o > 1.0f) return 0;
    float n = sqrtf(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    if (!(n > 0.0f)) return 0;
    float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    float R[3][3];
    R[0][0] = 1.0f - 2.0f * (y * y + z * z);
    R[0][1] = 2.0f * (x * y - w * z);
    R[0][2] = 2.0f * (x * z + w * y);
    R[1][0] = 2.0f * (x * y + w * z);
    R[1][1] = 1.0f - 2.0f * (x * x + z * z);
    R[1][2] = 2.0f * (y * z - w * x);
    R[2][0] = 2.0f * (x * z - w * y);
    R[2][1] = 2.0f * (y * z + w * x);
    R[2][2] = 1.0f - 2.0f * (x * x + y * y);
    float M[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) M[a][b] = R[a][b] * s[b];
    int idx = 0;
    for (int a = 0; a < 3; a++)
        for (int b = a; b < 3; b++)
            V[idx++] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];
    return 1;
}

/* Steps V1-V7: EWA projection. */
static void project(const float *mu, const float V6[6], float o, const ora_camera *cam, ora_proj *out) {
    const float *P = cam->w2c;
    memset(out, 0, sizeof(*out));
    out->o = o;
    float t[3];
    for (int a = 0; a < 3; a++)
        t[a] = ((P[4 * a + 0] * mu[0] + P[4 * a + 1] * mu[1]) + P[4 * a + 2] * mu[2]) + P[4 * a + 3];
    out->depth = t[2];
    if (!(t[2] > K_NEAR)) return;
    float u = t[0] / t[2], v = t[1] / t[2];
    out->mx = cam->fx * u + cam->cx;
    out->my = cam->fy * v + cam->cy;
    float j00 = cam->fx / t[2];
    float j02 = -(cam->fx * u) / t[2];
    float j11 = cam->fy / t[2];
    float j12 = -(cam->fy * v) / t[2];
    float Q[2][3];
    for (int b = 0; b < 3; b++) {
        Q[0][b] = j00 * P[0 * 4 + b] + j02 * P[2 * 4 + b];
        Q[1][b] = j11 * P[1 * 4 + b] + j12 * P[2 * 4 + b];
    }
    float Vm[3][3] = {{V6[0], V6[1], V6[2]}, {V6[1], V6[3], V6[4]}, {V6[2], V6[4], V6[5]}};
    float U[2][3];
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 3; b++)
            U[a][b] = (Q[a][0] * Vm[0][b] + Q[a][1] * Vm[1][b]) + Q[a][2] * Vm[2][b];
    float sxx = ((U[0][0] * Q[0][0] + U[0][1] * Q[0][1]) + U[0][2] * Q[0][2]) + K_LOWPASS;
    float sxy = (U[0][0] * Q[1][0] + U[0][1] * Q[1][1]) + U[0][2] * Q[1][2];
    float syy = ((U[1][0] * Q[1][0] + U[1][1] * Q[1][1]) + U[1][2] * Q[1][2]) + K_LOWPASS;
    out->sxx = sxx; out->sxy = sxy; out->syy = syy;
    float det = sxx * syy - sxy * sxy;
    if (!(det > 0.0f)) return;
    out->ca = syy / det;
    out->cb = -sxy / det;
    out->cc = sxx / det;
    float mid = 0.5f * (sxx + syy);
    float lam = mid + sqrtf(fmaxf(0.0f, mid * mid - det));
    out->r = 3.0f * sqrtf(lam);
    out->qa = out->ca * K_HALF_LOG2E;
    out->qb = out->cb * K_LOG2E_NEG;
    out->qc = out->cc * K_HALF_LOG2E;
    out->visible = 1;
}

/* One fragment test of Eq. 2 at pixel (x,y) (DESIGN.md §3 step PX).  Returns 1 and sets
 * *alpha when the Gaussian passes the support test, the y<=0 guard and alpha >= 1/255. */
static int fragment_alpha(const ora_proj *g, int x, int y, float *alpha) {
    float px = (float)x + 0.5f, py = (float)y + 0.5f;
    float dx = px - g->mx, dy = py - g->my;
    if (fabsf(dx) > g->r || fabsf(dy) > g->r) return 0;
    float q = fmaf(dx, fmaf(g->qa, dx, g->qb * dy), (g->qc * dy) * dy);
    if (q > 0.0f) return 0;
    float a = fminf(K_ACLAMP, g->o * ora_exp2_spec(q));
    if (a < K_AMIN) return 0;
    *alpha = a;
    return 1;
}

typedef struct { float depth; int64_t idx; } depth_key;

static int cmp_depth(const void *pa, const void *pb) {
    const depth_key *a = (const depth_key *)pa, *b = (const depth_key *)pb;
    if (a->depth < b->depth) return -1;
    if (a->depth > b->depth) return 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* ------------------------------------------------------------------------------------ */
/* Public entry points (ctypes).  Return 0 on success, negative on error; *err_index set. */

/* Activation + projection of every Gaussian for one camera (for projection pins).
 * out[G][16] = visible, depth, mx, my, sxx, sxy, syy, ca, cb, cc, r, qa, qb, qc, o, valid */
int ora_project(int64_t G, const float *means, const float *scales, const float *rots,
                const float *opac, const ora_camera *cam, float *out) {
    for (int64_t i = 0; i < G; i++) {
        float V[6];
        float *o = out + 16 * i;
        memset(o, 0, 16 * sizeof(float));
        if (!activate(rots + 4 * i, scales + 3 * i, opac[i], V)) continue;
        ora_proj p;
        project(means + 3 * i, V, opac[i], cam, &p);
        float vals[16] = {(float)p.visible, p.depth, p.mx, p.my, p.sxx, p.sxy, p.syy, p.ca, p.cb, p.cc,
                          p.r, p.qa, p.qb, p.qc, p.o, 1.0f};
        memcpy(o, vals, sizeof(vals));
    }
    return 0;
}

/* Splat one view Gaussian-major.  Per-pixel transmittance T (fp32) starts at 1.
 * Calls emit(i, pixel, e) for each fragment.  T_final [H*W] receives the final
 * transmittance.  Returns number of fragments, or -1 on invalid Gaussian (err_index). */
typedef void (*emit_fn)(void *ctx, int64_t i, int64_t pixel, float e);

static int64_t splat_view(int64_t G, const float *means, const ora_proj *proj, const ora_camera *cam,
                          float *T, unsigned char *done, emit_fn emit, void *ctx) {
    (void)means;
    const int W = cam->width, H = cam->height;
    depth_key *keys = (depth_key *)malloc(sizeof(depth_key) * (size_t)(G > 0 ? G : 1));
    int64_t nv = 0;
    for (int64_t i = 0; i < G; i++)
        if (proj[i].visible) { keys[nv].depth = proj[i].depth; keys[nv].idx = i; nv++; }
    qsort(keys, (size_t)nv, sizeof(depth_key), cmp_depth); /* (depth, index) order */
    for (int64_t p = 0; p < (int64_t)W * H; p++) { T[p] = 1.0f; done[p] = 0; }
    int64_t nfrag = 0;
    for (int64_t k = 0; k < nv; k++) {
        const ora_proj *g = &proj[keys[k].idx];
        /* conservative pixel range of the square support |x+0.5-mx| <= r (exact test below) */
        double pad = 2.0 + 1e-6 * (fabs((double)g->mx) + fabs((double)g->my) + (double)g->r);
        double x0d = floor((double)g->mx - (double)g->r - 0.5 - pad);
        double x1d = ceil((double)g->mx + (double)g->r - 0.5 + pad);
        double y0d = floor((double)g->my - (double)g->r - 0.5 - pad);
        double y1d = ceil((double)g->my + (double)g->r - 0.5 + pad);
        int x0 = x0d < 0 ? 0 : (x0d > W - 1 ? W : (int)x0d);
        int x1 = x1d > W - 1 ? W - 1 : (x1d < 0 ? -1 : (int)x1d);
        int y0 = y0d < 0 ? 0 : (y0d > H - 1 ? H : (int)y0d);
        int y1 = y1d > H - 1 ? H - 1 : (y1d < 0 ? -1 : (int)y1d);
        for (int y = y0; y <= y1; y++) {
            for (int x = x0; x <= x1; x++) {
                int64_t pix = (int64_t)y * W + x;
                if (done[pix]) continue;
                float a;
                if (!fragment_alpha(g, x, y, &a)) continue;
                float Tn = T[pix] * (1.0f - a);
                if (Tn < K_TMIN) { done[pix] = 1; continue; } /* pixel ends; no contribution */
                float e = a * T[pix];
                emit(ctx, keys[k].idx, pix, e);
                nfrag++;
                T[pix] = Tn;
            }
        }
    }
    free(keys);
    return nfrag;
}

static int prepare(int64_t G, const float *means, const float *scales, const float *rots,
                   const float *opac, const ora_camera *cam, ora_proj *proj, int64_t *err_index) {
    for (int64_t i = 0; i < G; i++) {
        float V[6];
        for (int k = 0; k < 3; k++)
            if (!isfinite(means[3 * i + k])) { *err_index = i; return -1; }
        if (!activate(rots + 4 * i, scales + 3 * i, opac[i], V)) { *err_index = i; return -1; }
        project(means + 3 * i, V, opac[i], cam, &proj[i]);
    }
    return 0;
}

typedef struct {
    int64_t cap, n;
    int64_t *pix, *gid;
    float *e;
} frag_list;

static void emit_list(void *ctx, int64_t i, int64_t pixel, float e) {
    frag_list *fl = (frag_list *)ctx;
    if (fl->n < fl->cap) { fl->pix[fl->n] = pixel; fl->gid[fl->n] = i; fl->e[fl->n] = e; }
    fl->n++;
}

/* Render one view's fragment list (pixel, gaussian, e) in emission order and T_final.
 * Returns the fragment count (may exceed cap: then only the first cap are stored). */
int64_t ora_render_view(int64_t G, const float *means, const float *scales, const float *rots,
                        const float *opac, const ora_camera *cam, float *T_final,
                        int64_t cap, int64_t *frag_pix, int64_t *frag_gid, float *frag_e,
                        int64_t *err_index) {
    ora_proj *proj = (ora_proj *)calloc((size_t)(G > 0 ? G : 1), sizeof(ora_proj));
    unsigned char *done = (unsigned char *)malloc((size_t)cam->width * cam->height);
    if (prepare(G, means, scales, rots, opac, cam, proj, err_index) < 0) { free(proj); free(done); return -1; }
    frag_list fl = {cap, 0, frag_pix, frag_gid, frag_e};
    int64_t n = splat_view(G, means, proj, cam, T_final, done, emit_list, &fl);
    free(proj); free(done);
    return n;
}

typedef struct {
    const uint32_t *ids;        /* region map of this view [H*W] */
    const uint32_t *atoms;      /* codes of this view [R][S] */
    const float *coefs;
    int32_t R, S, L;
    double *W, *Z;
    int64_t bad_region;         /* first pixel with id >= R (and != NONE), else -1 */
} agg_ctx;

/* Eq. 5 inner loop (Algorithm 1): w_i[j] += c_j * e_i(v,p); Z_i += e. */
static void emit_aggregate(void *vctx, int64_t i, int64_t pixel, float e) {
    agg_ctx *c = (agg_ctx *)vctx;
    c->Z[i] += (double)e;
    uint32_t rid = c->ids[pixel];
    if (rid == ORA_NONE) return;               /* unassigned pixel: no code */
    if (rid >= (uint32_t)c->R) { if (c->bad_region < 0) c->bad_region = pixel; return; }
    for (int s = 0; s < c->S; s++) {
        uint32_t a = c->atoms[(int64_t)rid * c->S + s];
        if (a == ORA_NONE) continue;           /* empty slot */
        float ce = c->coefs[(int64_t)rid * c->S + s] * e;  /* fp32 product */
        c->W[(int64_t)i * c->L + a] += (double)ce;
    }
}

/* Algorithm 1's per-pixel TopK(W_v(p)) applied to one region code: keep the K
 * largest coefficients (ties -> lower atom), no renormalisation; other slots emptied. */
static void truncate_code(uint32_t *atoms, float *coefs, int S, int K) {
    if (S <= K) return; /* already <= K-sparse: identity */
    for (int kept = 0; kept < K; kept++) {
        int best = -1;
        for (int s = kept; s < S; s++) {
            if (atoms[s] == ORA_NONE) continue;
            if (best < 0 || coefs[s] > coefs[best] || (coefs[s] == coefs[best] && atoms[s] < atoms[best]))
                best = s;
        }
        if (best < 0) break;
        uint32_t ta = atoms[kept]; float tc = coefs[kept];
        atoms[kept] = atoms[best]; coefs[kept] = coefs[best];
        atoms[best] = ta; coefs[best] = tc;
    }
    for (int s = K; s < S; s++) { atoms[s] = ORA_NONE; coefs[s] = 0.0f; }
}

/* Accumulate views into W [G][L] and Z [G] (fp64, caller-zeroed).
 * region_ids: [V][H][W]; codes for view v are rows code_row0[v] .. +num_regions[v].
 * view_frags[v] receives the contribution count of view v.
 * Errors: -2 bad Gaussian (err_index = i), -3 bad region id (err_index = view*H*W + pixel),
 *         -4 bad code (err_index = row*S + slot), -1 bad argument. */
int ora_uplift_accumulate(int64_t G, const float *means, const float *scales, const float *rots,
                          const float *opac, int32_t V, const ora_camera *cams,
                          const uint32_t *region_ids, const int64_t *code_row0,
                          const int32_t *num_regions, const uint32_t *code_atoms,
                          const float *code_coefs, int32_t S, int32_t L, int32_t K,
                          double *W, double *Z, int64_t *view_frags, int64_t *err_index) {
    if (K < 1 || K > L || S < 1 || L < 1) return -1;
    int64_t off = 0;
    for (int32_t v = 0; v < V; v++) {
        const ora_camera *cam = &cams[v];
        int64_t npx = (int64_t)cam->width * cam->height;
        int32_t R = num_regions[v];
        /* validate + truncate this view's codes (copy) */
        uint32_t *atoms = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(R > 0 ? R : 1) * S);
        float *coefs = (float *)malloc(sizeof(float) * (size_t)(R > 0 ? R : 1) * S);
        /* code_atoms == NULL: dense region features F_v(p) in R^L (Eq. 3, the dense
           uplift baseline): slot s is atom s, any finite value, no TopK truncation */
        const int dense = code_atoms == NULL;
        if (dense && S != L) { free(atoms); free(coefs); return -1; }
        for (int64_t j = 0; j < (int64_t)R * S; j++) {
            int64_t src = code_row0[v] * S + j;
            atoms[j] = dense ? (uint32_t)(j % S) : code_atoms[src];
            coefs[j] = code_coefs[src];
            if (atoms[j] != ORA_NONE &&
                (atoms[j] >= (uint32_t)L || !isfinite(coefs[j]) || (!dense && coefs[j] < 0.0f))) {
                *err_index = src; free(atoms); free(coefs); return -4;
            }
        }
        if (!dense)
            for (int32_t r = 0; r < R; r++) truncate_code(atoms + (int64_t)r * S, coefs + (int64_t)r * S, S, K);
        ora_proj *proj = (ora_proj *)calloc((size_t)(G > 0 ? G : 1), sizeof(ora_proj));
        float *T = (float *)malloc(sizeof(float) * (size_t)npx);
        unsigned char *done = (unsigned char *)malloc((size_t)npx);
        if (prepare(G, means, scales, rots, opac, cam, proj, err_index) < 0) {
            free(atoms); free(coefs); free(proj); free(T); free(done); return -2;
        }
        agg_ctx c = {region_ids + off, atoms, coefs, R, S, L, W, Z, -1};
        view_frags[v] = splat_view(G, means, proj, cam, T, done, emit_aggregate, &c);
        free(atoms); free(coefs); free(proj); free(T); free(done);
        if (c.bad_region >= 0) { *err_index = off + c.bad_region; return -3; }
        off += npx;
    }
    return 0;
}

/* Eq. 6 on one fp64 row: order (value desc, atom asc), keep the first K
 * entries with value > 0, divide by their fp64 sum; pad (NONE, 0). Returns #kept. */
int ora_topk_row(const double *w, int32_t L, int32_t K, uint32_t *atoms, double *coefs) {
    int32_t kept = 0;
    unsigned char *used = (unsigned char *)calloc((size_t)L, 1);
    for (int32_t k = 0; k < K; k++) {
        int32_t best = -1;
        for (int32_t a = 0; a < L; a++) {
            if (used[a] || !(w[a] > 0.0)) continue;
            if (best < 0 || w[a] > w[best]) best = a;  /* strict >: ties keep lower atom */
        }
        if (best < 0) break;
        used[best] = 1;
        atoms[kept] = (uint32_t)best;
        coefs[kept] = w[best];
        kept++;
    }
    free(used);
    double sum = 0.0;
    for (int32_t k = 0; k < kept; k++) sum += coefs[k];
    for (int32_t k = 0; k < kept; k++) coefs[k] /= sum;
    for (int32_t k = kept; k < K; k++) { atoms[k] = ORA_NONE; coefs[k] = 0.0; }
    return kept;
}

int ora_topk(int64_t G, const double *W, int32_t L, int32_t K, uint32_t *atoms, double *coefs) {
    for (int64_t i = 0; i < G; i++) ora_topk_row(W + i * L, L, K, atoms + i * K, coefs + i * K);
    return 0;
}

float ora_exp2_spec_vec(int64_t n, const float *y, float *out) {
    for (int64_t i = 0; i < n; i++) out[i] = ora_exp2_spec(y[i]);
    return 0.0f;
}
