/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product. See mfreg_oracle.h.
 *
 * Plain-C restatement of the reference hot path, written from the reference's
 * behaviour (citations are /root/reference/proj/<file>:<line>). Single-threaded:
 * the reference's results are thread-count invariant (README.md:53-55), so a
 * serial restatement of its fixed-order loops is bitwise equal to it.
 */
#include "mfreg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */
static char g_err[256];
enum { OK = 0, E_INVALID = 1, E_LOGIC = 2, E_OTHER = 3 };
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
const char* mport_last_error(void) { return g_err; }
void mport_set_threads(int n) { (void)n; }
int mport_thread_count(void) { return 1; }

/* ------------------------------------------------------------------- grid */
/* grid.hpp:16-45 — directions {-z,-y,-x,0,+x,+y,+z} */
enum { NEGZ = 0, NEGY, NEGX, CENTER, POSX, POSY, POSZ };
static int dir_axis(int d) {
    switch (d) {
    case NEGX: case POSX: return 0;
    case NEGY: case POSY: return 1;
    case NEGZ: case POSZ: return 2;
    default: return -1;
    }
}
static int dir_sign(int d) { return d < CENTER ? -1 : (d == CENTER ? 0 : 1); }
static int dir_opposite(int d) { return 6 - d; }

typedef struct {
    int64_t m[3];
    double h[3];
    int nodal;
} grid_t;

static int64_t g_count(const grid_t* g) { return g->m[0] * g->m[1] * g->m[2]; }
static double g_cellvol(const grid_t* g) { return g->h[0] * g->h[1] * g->h[2]; } /* grid.hpp:57 */
static double g_extent(const grid_t* g, int a) {                                 /* grid.hpp:59-62 */
    return g->nodal ? (double)(g->m[a] - 1) * g->h[a] : (double)g->m[a] * g->h[a];
}
static int64_t g_linear(const grid_t* g, int64_t i, int64_t j, int64_t k) {
    return i + j * g->m[0] + k * g->m[0] * g->m[1];
}
static void g_decompose(const grid_t* g, int64_t idx, int64_t c[3]) { /* grid.hpp:65-70 */
    c[0] = idx % g->m[0];
    c[1] = (idx / g->m[0]) % g->m[1];
    c[2] = idx / (g->m[0] * g->m[1]);
}
static int64_t g_neighbor(const grid_t* g, int64_t idx, int d) { /* grid.hpp:74-89 */
    if (d == CENTER) return idx;
    int64_t c[3];
    g_decompose(g, idx, c);
    const int a = dir_axis(d);
    int64_t v = c[a] + dir_sign(d);
    if (v < 0) v = 0;
    if (v > g->m[a] - 1) v = g->m[a] - 1;
    c[a] = v;
    return g_linear(g, c[0], c[1], c[2]);
}
static void g_point(const grid_t* g, int64_t idx, double p[3]) { /* grid.hpp:91-101 */
    int64_t c[3];
    g_decompose(g, idx, c);
    for (int a = 0; a < 3; ++a) {
        const double base = (double)c[a];
        p[a] = g->nodal ? base * g->h[a] : (base + 0.5) * g->h[a];
    }
}
static int g_validate(const grid_t* g) { /* grid.hpp:103-119 */
    for (int a = 0; a < 3; ++a) {
        if (g->m[a] < 1) return fail(E_INVALID, "GridDesc: all m components must be >= 1");
        if (!(g->h[a] > 0.0)) return fail(E_INVALID, "GridDesc: all h components must be > 0");
    }
    if (g->nodal)
        for (int a = 0; a < 3; ++a)
            if (g->m[a] < 2) return fail(E_INVALID, "GridDesc: nodal grids need >= 2 points per axis");
    return OK;
}
static grid_t image_grid(const int64_t* m, const double* h) {
    grid_t g = {{m[0], m[1], m[2]}, {h[0], h[1], h[2]}, 0};
    return g;
}
static grid_t nodal_grid(const int64_t* m, const double* h) {
    grid_t g = {{m[0], m[1], m[2]}, {h[0], h[1], h[2]}, 1};
    return g;
}
/* grid.hpp:131-146 */
static int make_deform_grid(const grid_t* img, const int64_t* pts, grid_t* out) {
    out->nodal = 1;
    for (int a = 0; a < 3; ++a) {
        out->m[a] = pts[a];
        if (pts[a] < 2) return fail(E_INVALID, "deformation grid needs >= 2 points per axis");
        if (pts[a] - 1 > img->m[a]) return fail(E_INVALID, "deformation grid finer than image grid");
        out->h[a] = g_extent(img, a) / (double)(pts[a] - 1);
    }
    return OK;
}

/* ------------------------------------------------------------ reductions */
/* parallel.cpp:51-73 — 4096-element chunks summed sequentially, partials in chunk order */
#define CHUNK 4096
typedef double (*term_fn)(int64_t i, const void* ctx);
static double chunked_sum(int64_t n, term_fn term, const void* ctx) {
    if (n <= 0) return 0.0;
    const int64_t nchunks = (n + CHUNK - 1) / CHUNK;
    double total = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t lo = c * CHUNK;
        const int64_t hi = (lo + CHUNK < n) ? lo + CHUNK : n;
        double s = 0.0;
        for (int64_t i = lo; i < hi; ++i) s += term(i, ctx);
        total += s;
    }
    return total;
}
typedef struct { const double* a; const double* b; } dot_ctx;
static double dot_term(int64_t i, const void* c) {
    const dot_ctx* d = (const dot_ctx*)c;
    return d->a[i] * d->b[i];
}
static double vec_dot(const double* a, const double* b, int64_t n) { /* optimizer.cpp:12-19 */
    dot_ctx c = {a, b};
    return chunked_sum(n, dot_term, &c);
}
static double vec_norm(const double* a, int64_t n) { return sqrt(vec_dot(a, a, n)); } /* :21 */
static double vec_inf_norm(const double* a, int64_t n) {                                /* :23-29 */
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double x = fabs(a[i]);
        m = (m < x) ? x : m;
    }
    return m;
}

/* ------------------------------------------------------------------ image */
static double sample_or_zero(const double* t, const grid_t* g, int64_t i, int64_t j, int64_t k) {
    if (i < 0 || j < 0 || k < 0 || i >= g->m[0] || j >= g->m[1] || k >= g->m[2]) return 0.0;
    return t[g_linear(g, i, j, k)]; /* volume.cpp:19-25 */
}

/* volume.cpp:29-74 — trilinear, Dirichlet zeros, ties to the lower cell */
static void interpolate(const double* t, const grid_t* g, const double p[3], double* value, double grad[3]) {
    int64_t base[3];
    double f[3];
    for (int a = 0; a < 3; ++a) {
        const double s = p[a] / g->h[a] - 0.5;
        const double c = ceil(s);
        base[a] = (int64_t)c - 1;
        f[a] = s - (double)base[a];
    }
    double v[2][2][2];
    for (int gg = 0; gg < 2; ++gg)
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) v[gg][b][a] = sample_or_zero(t, g, base[0] + a, base[1] + b, base[2] + gg);
    const double fx = f[0], fy = f[1], fz = f[2];
    double cx[2][2], dx[2][2];
    for (int gg = 0; gg < 2; ++gg)
        for (int b = 0; b < 2; ++b) {
            cx[gg][b] = v[gg][b][0] * (1.0 - fx) + v[gg][b][1] * fx;
            dx[gg][b] = v[gg][b][1] - v[gg][b][0];
        }
    double cy[2], dyv[2], dxv[2];
    for (int gg = 0; gg < 2; ++gg) {
        cy[gg] = cx[gg][0] * (1.0 - fy) + cx[gg][1] * fy;
        dyv[gg] = cx[gg][1] - cx[gg][0];
        dxv[gg] = dx[gg][0] * (1.0 - fy) + dx[gg][1] * fy;
    }
    *value = cy[0] * (1.0 - fz) + cy[1] * fz;
    const double gx = dxv[0] * (1.0 - fz) + dxv[1] * fz;
    const double gy = dyv[0] * (1.0 - fz) + dyv[1] * fz;
    const double gz = cy[1] - cy[0];
    grad[0] = gx / g->h[0];
    grad[1] = gy / g->h[1];
    grad[2] = gz / g->h[2];
}

/* volume.cpp:76-94 */
static void sample_deformed(const double* t, const grid_t* g, const double* pts, int64_t n, double* values,
                            double* partials) {
    for (int64_t i = 0; i < n; ++i) {
        const double p[3] = {pts[i], pts[n + i], pts[2 * n + i]};
        double gr[3];
        interpolate(t, g, p, &values[i], gr);
        partials[i] = gr[0];
        partials[n + i] = gr[1];
        partials[2 * n + i] = gr[2];
    }
}

/* volume.cpp:96-109 — backward x,y,z then forward x,y,z, clamped neighbours */
static void discrete_gradient(const double* data, const grid_t* g, int64_t i, double r[6]) {
    static const int neg[3] = {NEGX, NEGY, NEGZ};
    static const int pos[3] = {POSX, POSY, POSZ};
    const double vi = data[i];
    for (int a = 0; a < 3; ++a) {
        const double h = g->h[a];
        r[a] = (vi - data[g_neighbor(g, i, neg[a])]) / h;
        r[a + 3] = (data[g_neighbor(g, i, pos[a])] - vi) / h;
    }
}

/* volume.cpp:115-121 */
static double eps_norm(const double g[6], double eps) {
    double s = 0.0;
    for (int k = 0; k < 6; ++k) s += g[k] * g[k];
    return sqrt(0.5 * s + eps * eps);
}

/* volume.cpp:123-160 */
static int downsample(const double* v, const grid_t* g, double* out, grid_t* c) {
    for (int a = 0; a < 3; ++a)
        if (g->m[a] < 2) return fail(E_INVALID, "downsample: all axes must have m >= 2");
    c->nodal = 0;
    for (int a = 0; a < 3; ++a) {
        c->m[a] = (g->m[a] + 1) / 2;
        c->h[a] = 2.0 * g->h[a];
    }
    if (!out) return OK;
    for (int64_t k = 0; k < c->m[2]; ++k)
        for (int64_t j = 0; j < c->m[1]; ++j)
            for (int64_t i = 0; i < c->m[0]; ++i) {
                double sum = 0.0;
                int cnt = 0;
                for (int64_t dz = 0; dz < 2; ++dz)
                    for (int64_t dy = 0; dy < 2; ++dy)
                        for (int64_t dx = 0; dx < 2; ++dx) {
                            const int64_t fi = 2 * i + dx, fj = 2 * j + dy, fk = 2 * k + dz;
                            if (fi < g->m[0] && fj < g->m[1] && fk < g->m[2]) {
                                sum += v[g_linear(g, fi, fj, fk)];
                                ++cnt;
                            }
                        }
                out[g_linear(c, i, j, k)] = sum / cnt;
            }
    return OK;
}

/* --------------------------------------------------------------- transfer */
typedef struct {
    grid_t source, target;
    int64_t* base[3];
    double* rem[3];
} plan_t;

static void plan_free(plan_t* p) {
    for (int a = 0; a < 3; ++a) {
        free(p->base[a]);
        free(p->rem[a]);
        p->base[a] = NULL;
        p->rem[a] = NULL;
    }
}

/* transfer.cpp:11-47 */
static int make_plan(const grid_t* src, const grid_t* tgt, plan_t* plan) {
    memset(plan, 0, sizeof *plan);
    if (!src->nodal || tgt->nodal)
        return fail(E_INVALID, "transfer plan needs nodal source and cell-centered target");
    int rc = g_validate(src);
    if (rc) return rc;
    if ((rc = g_validate(tgt))) return rc;
    plan->source = *src;
    plan->target = *tgt;
    for (int a = 0; a < 3; ++a) {
        const int64_t mt = tgt->m[a], ms = src->m[a];
        plan->base[a] = (int64_t*)malloc(sizeof(int64_t) * mt);
        plan->rem[a] = (double*)malloc(sizeof(double) * mt);
        for (int64_t k = 0; k < mt; ++k) {
            const double c = ((double)k + 0.5) * (double)(ms - 1) / (double)mt;
            int64_t b = (int64_t)floor(c);
            if (b < 0) b = 0;
            if (b > ms - 2) b = ms - 2;
            plan->base[a][k] = b;
            plan->rem[a][k] = c - (double)b;
            if (plan->rem[a][k] < 0.0 || plan->rem[a][k] > 1.0) {
                plan_free(plan);
                return fail(E_INVALID, "transfer plan: coverage invariant violated");
            }
        }
    }
    return OK;
}

/* transfer.cpp:49-86 — acc += ((wx*wy)*wz)*y in (g,b,a) order */
static void transfer_apply(const plan_t* plan, const double* y, double* out) {
    const grid_t* t = &plan->target;
    const int64_t nt = g_count(t), ns = g_count(&plan->source);
    const int64_t* sm = plan->source.m;
    for (int64_t i = 0; i < nt; ++i) {
        int64_t c[3];
        g_decompose(t, i, c);
        const int64_t bx = plan->base[0][c[0]], by = plan->base[1][c[1]], bz = plan->base[2][c[2]];
        const double rx = plan->rem[0][c[0]], ry = plan->rem[1][c[1]], rz = plan->rem[2][c[2]];
        const double wx[2] = {1.0 - rx, rx}, wy[2] = {1.0 - ry, ry}, wz[2] = {1.0 - rz, rz};
        for (int d = 0; d < 3; ++d) {
            const double* yd = y + d * ns;
            double acc = 0.0;
            for (int g = 0; g < 2; ++g)
                for (int b = 0; b < 2; ++b)
                    for (int a = 0; a < 2; ++a) {
                        const int64_t src = (bx + a) + (by + b) * sm[0] + (bz + g) * sm[0] * sm[1];
                        acc += wx[a] * wy[b] * wz[g] * yd[src];
                    }
            out[d * nt + i] = acc;
        }
    }
}

/* transfer.cpp:92-150 — odd deformation z-slabs first, then even; inside a slab
 * image planes ascending, then rows, then columns. */
static void transfer_apply_transpose(const plan_t* plan, const double* w, double* out) {
    const grid_t* t = &plan->target;
    const int64_t nt = g_count(t), ns = g_count(&plan->source);
    const int64_t* tm = t->m;
    const int64_t* sm = plan->source.m;
    memset(out, 0, sizeof(double) * 3 * ns);
    const int64_t nslabs = sm[2] - 1;
    for (int phase = 0; phase < 2; ++phase) {
        const int64_t first = phase == 0 ? 1 : 0;
        for (int64_t slab = first; slab < nslabs; slab += 2) {
            for (int64_t kz = 0; kz < tm[2]; ++kz) {
                if (plan->base[2][kz] != slab) continue; /* slab_planes, transfer.cpp:41-45 */
                const int64_t bz = plan->base[2][kz];
                const double rz = plan->rem[2][kz];
                const double wzv[2] = {1.0 - rz, rz};
                for (int64_t ky = 0; ky < tm[1]; ++ky) {
                    const int64_t by = plan->base[1][ky];
                    const double ry = plan->rem[1][ky];
                    const double wyv[2] = {1.0 - ry, ry};
                    for (int64_t kx = 0; kx < tm[0]; ++kx) {
                        const int64_t bx = plan->base[0][kx];
                        const double rx = plan->rem[0][kx];
                        const double wxv[2] = {1.0 - rx, rx};
                        const int64_t ti = kx + ky * tm[0] + kz * tm[0] * tm[1];
                        for (int d = 0; d < 3; ++d) {
                            const double v = w[d * nt + ti];
                            double* od = out + d * ns;
                            for (int g = 0; g < 2; ++g)
                                for (int b = 0; b < 2; ++b)
                                    for (int a = 0; a < 2; ++a) {
                                        const int64_t dst = (bx + a) + (by + b) * sm[0] + (bz + g) * sm[0] * sm[1];
                                        od[dst] += wxv[a] * wyv[b] * wzv[g] * v;
                                    }
                        }
                    }
                }
            }
        }
    }
}

/* -------------------------------------------------------------------- NGF */
typedef struct {
    grid_t g;
    double tau, rho;
    double* ref;       /* n */
    double* ref_grads; /* 6n, [i*6+c] */
    double* ref_norms; /* n */
    /* workspace, ngf.hpp:31-37 */
    double* values;    /* n */
    double* partials;  /* 3n component-major */
    double* tpl_grads; /* 6n, [i*6+c] */
    double* residual;  /* n */
    double* inv1;      /* n */
    double* inv2;      /* n */
} ngf_t;

static void ngf_free(ngf_t* c) {
    if (!c) return;
    free(c->ref); free(c->ref_grads); free(c->ref_norms); free(c->values); free(c->partials);
    free(c->tpl_grads); free(c->residual); free(c->inv1); free(c->inv2);
    free(c);
}

/* ngf.cpp:167-183 */
static ngf_t* ngf_new(const double* ref, const grid_t* g, double tau, double rho, int* rc) {
    if (!(rho > 0.0)) {
        *rc = fail(E_INVALID, "NGF: rho must be > 0");
        return NULL;
    }
    ngf_t* c = (ngf_t*)calloc(1, sizeof(ngf_t));
    const int64_t n = g_count(g);
    c->g = *g;
    c->tau = tau;
    c->rho = rho;
    c->ref = (double*)malloc(sizeof(double) * n);
    memcpy(c->ref, ref, sizeof(double) * n);
    c->ref_grads = (double*)malloc(sizeof(double) * 6 * n);
    c->ref_norms = (double*)malloc(sizeof(double) * n);
    c->values = (double*)calloc(n, sizeof(double));
    c->partials = (double*)calloc(3 * n, sizeof(double));
    c->tpl_grads = (double*)calloc(6 * n, sizeof(double));
    c->residual = (double*)calloc(n, sizeof(double));
    c->inv1 = (double*)calloc(n, sizeof(double));
    c->inv2 = (double*)calloc(n, sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        discrete_gradient(c->ref, g, i, &c->ref_grads[6 * i]);
        c->ref_norms[i] = eps_norm(&c->ref_grads[6 * i], rho);
    }
    *rc = OK;
    return c;
}

/* ngf.cpp:185-214 */
static int ngf_populate(ngf_t* c, const double* tpl, const double* pts) {
    if (!(c->tau > 0.0) || !(c->rho > 0.0)) return fail(E_INVALID, "NGF: tau and rho must be > 0");
    const grid_t* g = &c->g;
    const int64_t n = g_count(g);
    sample_deformed(tpl, g, pts, n, c->values, c->partials);
    const double taurho = c->tau * c->rho;
    for (int64_t i = 0; i < n; ++i) {
        double* gt = &c->tpl_grads[6 * i];
        const double* gr = &c->ref_grads[6 * i];
        discrete_gradient(c->values, g, i, gt);
        const double tn = eps_norm(gt, c->tau);
        const double rn = c->ref_norms[i];
        double num = taurho;
        for (int k = 0; k < 6; ++k) num += 0.5 * gt[k] * gr[k];
        c->inv1[i] = 1.0 / (tn * rn);
        c->inv2[i] = num / (tn * tn * tn * rn);
        c->residual[i] = num * c->inv1[i];
    }
    return OK;
}

/* ngf.cpp:14-26 */
static int64_t dir_offset(int d, const grid_t* g) {
    switch (d) {
    case NEGZ: return -g->m[0] * g->m[1];
    case NEGY: return -g->m[0];
    case NEGX: return -1;
    case CENTER: return 0;
    case POSX: return 1;
    case POSY: return g->m[0];
    case POSZ: return g->m[0] * g->m[1];
    }
    return 0;
}

/* ngf.cpp:28-33 */
static void hhat(const grid_t* g, double hh[3]) {
    for (int a = 0; a < 3; ++a) hh[a] = 1.0 / (2.0 * g->h[a] * g->h[a]);
}

/* ngf.cpp:39-49 */
static double rho_dir(const ngf_t* c, int64_t i, int k) {
    const int a = dir_axis(k);
    const int sgn = dir_sign(k);
    const int comp = sgn > 0 ? a + 3 : a;
    const double h = c->g.h[a];
    const double dR = sgn * h * c->ref_grads[6 * i + comp];
    const double dT = sgn * h * c->tpl_grads[6 * i + comp];
    return dR * c->inv1[i] - dT * c->inv2[i];
}

/* ngf.cpp:51-64 */
static double rho_hat(const ngf_t* c, int64_t i, int k, const double hh[3]) {
    if (k == CENTER) {
        double s = 0.0;
        for (int d = 0; d < 7; ++d) {
            if (d == CENTER) continue;
            s -= hh[dir_axis(d)] * rho_dir(c, i, d);
        }
        return s;
    }
    return hh[dir_axis(k)] * rho_dir(c, i, k);
}

static double value_term(int64_t i, const void* ctx) {
    const double r = ((const ngf_t*)ctx)->residual[i];
    return 1.0 - r * r;
}
/* ngf.cpp:225-231 */
static double ngf_value(const ngf_t* c) {
    const double hbar = g_cellvol(&c->g);
    return hbar * chunked_sum(g_count(&c->g), value_term, c);
}

/* ngf.cpp:66-103 (Alg. 4.1) */
static void ngf_gradient(const ngf_t* c, double* out) {
    const grid_t* g = &c->g;
    const int64_t n = g_count(g);
    double hh[3];
    hhat(g, hh);
    const double scale = -2.0 * g_cellvol(g);
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < 7; ++k) {
            const int64_t j = i + dir_offset(k, g);
            if (j < 0 || j >= n) continue;
            acc += c->residual[j] * rho_hat(c, j, dir_opposite(k), hh);
        }
        const double s = scale * acc;
        out[i] = s * c->partials[i];
        out[n + i] = s * c->partials[n + i];
        out[2 * n + i] = s * c->partials[2 * n + i];
    }
}

/* ngf.cpp:267-300 — kappa ascending (std::map order), pairs in (da, db) insertion order */
typedef struct {
    int nentries;
    int64_t kappa[49];
    int npairs[49];
    int pa[49][49], pb[49][49];
} offset_table_t;

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

static int make_offset_table(const grid_t* g, offset_table_t* t) {
    int64_t ks[49];
    int nk = 0;
    for (int da = 0; da < 7; ++da)
        for (int db = 0; db < 7; ++db) ks[nk++] = dir_offset(db, g) - dir_offset(da, g);
    qsort(ks, 49, sizeof(int64_t), cmp_i64);
    t->nentries = 0;
    for (int q = 0; q < 49; ++q)
        if (q == 0 || ks[q] != ks[q - 1]) t->kappa[t->nentries++] = ks[q];
    for (int e = 0; e < t->nentries; ++e) {
        t->npairs[e] = 0;
        for (int da = 0; da < 7; ++da)
            for (int db = 0; db < 7; ++db)
                if (dir_offset(db, g) - dir_offset(da, g) == t->kappa[e]) {
                    t->pa[e][t->npairs[e]] = da;
                    t->pb[e][t->npairs[e]] = db;
                    ++t->npairs[e];
                }
    }
    if (t->nentries == 25) {
        const int64_t m1 = g->m[0], m12 = g->m[0] * g->m[1];
        int64_t ex[25] = {-2 * m12, -m12 - m1, -m12 - 1, -m12, -m12 + 1, -m12 + m1, -2 * m1, -m1 - 1, -m1,
                          -m1 + 1,  -2,        -1,       0,    1,        2,         m1 - 1,  m1,      m1 + 1,
                          2 * m1,   m12 - m1,  m12 - 1,  m12,  m12 + 1,  m12 + m1,  2 * m12};
        qsort(ex, 25, sizeof(int64_t), cmp_i64);
        for (int q = 0; q < 25; ++q)
            if (t->kappa[q] != ex[q]) return fail(E_LOGIC, "offset table mismatch against closed-form list");
    }
    return OK;
}

/* ngf.cpp:105-163 (Alg. 4.2) — closed-form 25-offset GN Hessian-vector product */
static int ngf_hessian_vec(const ngf_t* c, const double* p, double* out) {
    const grid_t* g = &c->g;
    const int64_t n = g_count(g);
    offset_table_t tab;
    int rc = make_offset_table(g, &tab);
    if (rc) return rc;
    double hh[3];
    hhat(g, hh);
    const double scale = 2.0 * g_cellvol(g);
    const double *px = p, *py = p + n, *pz = p + 2 * n;
    const double *d0 = c->partials, *d1 = c->partials + n, *d2 = c->partials + 2 * n;
    for (int64_t i = 0; i < n; ++i) {
        double qx = 0.0, qy = 0.0, qz = 0.0;
        for (int e = 0; e < tab.nentries; ++e) {
            const int64_t ti = i + tab.kappa[e];
            if (ti < 0 || ti >= n) continue;
            double drdr = 0.0;
            for (int q = 0; q < tab.npairs[e]; ++q) {
                const int da = tab.pa[e][q], db = tab.pb[e][q];
                const int64_t t = i + dir_offset(db, g);
                if (t < 0 || t >= n) continue;
                drdr += rho_hat(c, t, dir_opposite(da), hh) * rho_hat(c, t, dir_opposite(db), hh);
            }
            const double s = d0[ti] * px[ti] + d1[ti] * py[ti] + d2[ti] * pz[ti];
            const double cc = drdr * s;
            qx += cc * d0[i];
            qy += cc * d1[i];
            qz += cc * d2[i];
        }
        out[i] = scale * qx;
        out[n + i] = scale * qy;
        out[2 * n + i] = scale * qz;
    }
    return OK;
}

/* -------------------------------------------------------------- curvature */
/* curvature.cpp:9-21 */
static double laplacian(const double* u, const grid_t* g, int64_t i) {
    static const int neg[3] = {NEGX, NEGY, NEGZ};
    static const int pos[3] = {POSX, POSY, POSZ};
    const double ui = u[i];
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double h = g->h[a];
        s += (u[g_neighbor(g, i, neg[a])] - 2.0 * ui + u[g_neighbor(g, i, pos[a])]) / (h * h);
    }
    return s;
}
typedef struct { const double* u; const grid_t* g; } lap_ctx;
static double lap_sq_term(int64_t i, const void* c) {
    const lap_ctx* l = (const lap_ctx*)c;
    const double v = laplacian(l->u, l->g, i);
    return v * v;
}
/* curvature.cpp:35-49 */
static double curvature_value(const double* u, const grid_t* g) {
    const int64_t n = g_count(g);
    double total = 0.0;
    for (int d = 0; d < 3; ++d) {
        lap_ctx c = {u + d * n, g};
        total += chunked_sum(n, lap_sq_term, &c);
    }
    return g_cellvol(g) * total;
}
/* curvature.cpp:53-72 — 2 h^y Lap(Lap v) per component, two passes via scratch */
static void biharmonic(const double* v, const grid_t* g, double* scratch, double* out) {
    const int64_t n = g_count(g);
    const double scale = 2.0 * g_cellvol(g);
    for (int d = 0; d < 3; ++d) {
        for (int64_t i = 0; i < n; ++i) scratch[i] = laplacian(v + d * n, g, i);
        for (int64_t i = 0; i < n; ++i) out[d * n + i] = scale * laplacian(scratch, g, i);
    }
}

/* -------------------------------------------------------------- objective */
typedef struct {
    grid_t img, dg;
    double alpha;
    double* tpl;
    ngf_t* ngf;
    plan_t plan;
    double last_distance, last_regularizer;
    double *yhat, *dist_grad, *u, *reg_grad, *scratch, *php, *hphp, *xid;
} obj_t;

static void obj_free(obj_t* o) {
    if (!o) return;
    ngf_free(o->ngf);
    plan_free(&o->plan);
    free(o->tpl); free(o->yhat); free(o->dist_grad); free(o->u); free(o->reg_grad);
    free(o->scratch); free(o->php); free(o->hphp); free(o->xid);
    free(o);
}
static int64_t obj_dof(const obj_t* o) { return 3 * g_count(&o->dg); }
static double obj_min_spacing(const obj_t* o) { /* optimizer.hpp:68-70 */
    double m = o->dg.h[0];
    if (o->dg.h[1] < m) m = o->dg.h[1];
    if (o->dg.h[2] < m) m = o->dg.h[2];
    return m;
}

/* optimizer.cpp:31-62 */
static obj_t* obj_new(const double* ref, const double* tpl, const grid_t* img, const grid_t* dg, double tau,
                      double rho, double alpha, int* rc) {
    obj_t* o = (obj_t*)calloc(1, sizeof(obj_t));
    o->img = *img;
    o->dg = *dg;
    o->alpha = alpha;
    const int64_t n = g_count(img), ny = g_count(dg);
    o->ngf = ngf_new(ref, img, tau, rho, rc);
    if (*rc) { obj_free(o); return NULL; }
    if ((*rc = make_plan(dg, img, &o->plan))) { obj_free(o); return NULL; }
    o->tpl = (double*)malloc(sizeof(double) * n);
    memcpy(o->tpl, tpl, sizeof(double) * n);
    o->yhat = (double*)calloc(3 * n, sizeof(double));
    o->dist_grad = (double*)calloc(3 * n, sizeof(double));
    o->php = (double*)calloc(3 * n, sizeof(double));
    o->hphp = (double*)calloc(3 * n, sizeof(double));
    o->u = (double*)calloc(3 * ny, sizeof(double));
    o->reg_grad = (double*)calloc(3 * ny, sizeof(double));
    o->scratch = (double*)calloc(ny, sizeof(double));
    o->xid = (double*)calloc(3 * ny, sizeof(double));
    for (int64_t i = 0; i < ny; ++i) {
        double p[3];
        g_point(dg, i, p);
        for (int d = 0; d < 3; ++d) o->xid[d * ny + i] = p[d];
    }
    return o;
}

/* optimizer.cpp:64-92 */
static double obj_eval(obj_t* o, const double* y, double* grad) {
    const int64_t nd = obj_dof(o), ny = g_count(&o->dg);
    transfer_apply(&o->plan, y, o->yhat);
    ngf_populate(o->ngf, o->tpl, o->yhat);
    o->last_distance = ngf_value(o->ngf);
    for (int64_t i = 0; i < nd; ++i) o->u[i] = y[i] - o->xid[i];
    o->last_regularizer = o->alpha * curvature_value(o->u, &o->dg);
    if (grad) {
        ngf_gradient(o->ngf, o->dist_grad);
        transfer_apply_transpose(&o->plan, o->dist_grad, grad);
        if (o->alpha != 0.0) {
            biharmonic(o->u, &o->dg, o->scratch, o->reg_grad);
            for (int64_t i = 0; i < nd; ++i) grad[i] += o->alpha * o->reg_grad[i];
        }
    }
    (void)ny;
    return o->last_distance + o->last_regularizer;
}

/* optimizer.cpp:94-104 */
static void obj_gn_hv(obj_t* o, const double* p, double* q) {
    const int64_t nd = obj_dof(o);
    transfer_apply(&o->plan, p, o->php);
    ngf_hessian_vec(o->ngf, o->php, o->hphp);
    transfer_apply_transpose(&o->plan, o->hphp, q);
    if (o->alpha != 0.0) {
        biharmonic(p, &o->dg, o->scratch, o->reg_grad);
        for (int64_t i = 0; i < nd; ++i) q[i] += o->alpha * o->reg_grad[i];
    }
}

/* optimizer.cpp:106-111 */
static void obj_seed_hv(obj_t* o, const double* p, double gamma, double* q) {
    const int64_t nd = obj_dof(o);
    biharmonic(p, &o->dg, o->scratch, q);
    for (int64_t i = 0; i < nd; ++i) q[i] += gamma * p[i];
}

/* --------------------------------------------------------------- solvers */
typedef struct {
    obj_t* o;
    int seed;
    double gamma;
} op_t;
static void op_apply(const op_t* op, const double* v, double* out) {
    if (op->seed) obj_seed_hv(op->o, v, op->gamma, out);
    else obj_gn_hv(op->o, v, out);
}

/* optimizer.cpp:113-154 — plain CG, x0 = 0 */
static void cg_solve(const op_t* op, const double* b, int64_t n, int max_iters, double rel_tol, double* x,
                     int* iters, double* relres, int* breakdown) {
    memset(x, 0, sizeof(double) * n);
    *iters = 0;
    *relres = 0.0;
    *breakdown = 0;
    const double bnorm = vec_norm(b, n);
    if (bnorm == 0.0) return;
    double* r = (double*)malloc(sizeof(double) * n);
    double* p = (double*)malloc(sizeof(double) * n);
    double* ap = (double*)calloc(n, sizeof(double));
    memcpy(r, b, sizeof(double) * n);
    memcpy(p, b, sizeof(double) * n);
    double rr = vec_dot(r, r, n);
    for (int it = 0; it < max_iters; ++it) {
        op_apply(op, p, ap);
        const double pap = vec_dot(p, ap, n);
        if (!isfinite(pap) || pap <= 0.0) {
            *breakdown = !isfinite(pap);
            break;
        }
        const double alpha = rr / pap;
        for (int64_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * ap[i];
        }
        ++*iters;
        const double rr_new = vec_dot(r, r, n);
        *relres = sqrt(rr_new) / bnorm;
        if (!isfinite(rr_new)) {
            *breakdown = 1;
            break;
        }
        if (*relres <= rel_tol) break;
        const double beta = rr_new / rr;
        for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rr = rr_new;
    }
    free(r);
    free(p);
    free(ap);
}

/* optimizer.cpp:156-175 — phi(eta) = J(y + eta d), value-only eval */
static int armijo(obj_t* o, const double* y, const double* dir, double* y_trial, int64_t n, double f0,
                  double gdotd, const mport_opt_config* cfg, double eta0, double* eta_out) {
    if (!(gdotd < 0.0)) return 0;
    double eta = eta0;
    for (int k = 0; k <= cfg->max_backtracks; ++k) {
        for (int64_t i = 0; i < n; ++i) y_trial[i] = y[i] + eta * dir[i];
        const double f = obj_eval(o, y_trial, NULL);
        if (isfinite(f) && f <= f0 + cfg->c1 * eta * gdotd) {
            *eta_out = eta;
            return 1;
        }
        eta *= cfg->beta;
    }
    return 0;
}

/* optimizer.cpp:188-200 */
static int should_stop(const mport_opt_config* cfg, double g0, double min_hy, double j_prev, double j_cur,
                       double gnorm, double step_inf) {
    if (gnorm <= cfg->tol_grad * g0) return 1;
    const double aj = fabs(j_prev);
    if (fabs(j_prev - j_cur) <= cfg->tol_rel_j * (1.0 < aj ? aj : 1.0)) return 1;
    if (step_inf <= cfg->tol_step * min_hy) return 1;
    return 0;
}

static void push_rec(mport_iter_record* tr, int cap, int* nt, const mport_iter_record* r) {
    if (*nt < cap) tr[*nt] = *r;
    ++*nt;
}

/* optimizer.cpp:202-268 + 392-407 — Gauss-Newton descent loop */
static void gauss_newton(obj_t* o, const double* y0, const mport_opt_config* cfg, double* y,
                         mport_iter_record* tr, int cap, int* nt, int* lsf) {
    const int64_t n = obj_dof(o);
    memcpy(y, y0, sizeof(double) * n);
    *nt = 0;
    *lsf = 0;
    if (cfg->max_iters <= 0) return;
    double* grad = (double*)calloc(n, sizeof(double));
    double* dir = (double*)calloc(n, sizeof(double));
    double* yt = (double*)calloc(n, sizeof(double));
    double* b = (double*)calloc(n, sizeof(double));
    double j = obj_eval(o, y, grad);
    const double g0 = vec_norm(grad, n);
    const double min_hy = obj_min_spacing(o);
    op_t op = {o, 0, 0.0};
    for (int it = 0; it < cfg->max_iters; ++it) {
        mport_iter_record rec = {it, 0, j, o->last_distance, o->last_regularizer, vec_norm(grad, n), 0.0};
        if (rec.grad_norm <= cfg->tol_grad * g0) {
            push_rec(tr, cap, nt, &rec);
            break;
        }
        for (int64_t i = 0; i < n; ++i) b[i] = -grad[i];
        int iters, brk;
        double relres;
        cg_solve(&op, b, n, cfg->cg_max_iters, cfg->cg_rel_tol, dir, &iters, &relres, &brk);
        rec.cg_iters = iters;
        const double gdotd = vec_dot(grad, dir, n);
        const double dinf = vec_inf_norm(dir, n);
        double eta0 = 1.0;
        if (dinf > 0.0) {
            const double q = min_hy / dinf;
            eta0 = q < 1.0 ? q : 1.0;
        }
        double eta = 0.0;
        if (!armijo(o, y, dir, yt, n, j, gdotd, cfg, eta0, &eta)) {
            *lsf = 1;
            push_rec(tr, cap, nt, &rec);
            break;
        }
        rec.step = eta;
        const double j_prev = j;
        for (int64_t i = 0; i < n; ++i) y[i] += eta * dir[i];
        double step_inf = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double s = fabs(eta * dir[i]);
            step_inf = step_inf < s ? s : step_inf;
        }
        j = obj_eval(o, y, grad);
        push_rec(tr, cap, nt, &rec);
        if (should_stop(cfg, g0, min_hy, j_prev, j, vec_norm(grad, n), step_inf)) break;
    }
    free(grad); free(dir); free(yt); free(b);
}

/* optimizer.cpp:272-390 — L-BFGS, two-loop with H0 = Hess(S) + gamma I via CG */
static void lbfgs(obj_t* o, const double* y0, const mport_opt_config* cfg, double* y, mport_iter_record* tr,
                  int cap, int* nt, int* lsf) {
    const int64_t n = obj_dof(o);
    const double gamma = cfg->gamma >= 0.0 ? cfg->gamma : 1e-3 * (1.0 < o->alpha ? o->alpha : 1.0);
    const int hist_cap = cfg->lbfgs_history > 1 ? cfg->lbfgs_history : 1;
    double** hs = (double**)calloc(hist_cap + 1, sizeof(double*));
    double** hy = (double**)calloc(hist_cap + 1, sizeof(double*));
    double* hrho = (double*)calloc(hist_cap + 1, sizeof(double));
    int hn = 0;
    memcpy(y, y0, sizeof(double) * n);
    *nt = 0;
    *lsf = 0;
    if (cfg->max_iters <= 0) { free(hs); free(hy); free(hrho); return; }
    double* grad = (double*)calloc(n, sizeof(double));
    double* gnew = (double*)calloc(n, sizeof(double));
    double* dir = (double*)calloc(n, sizeof(double));
    double* yt = (double*)calloc(n, sizeof(double));
    double* q = (double*)calloc(n, sizeof(double));
    double* r = (double*)calloc(n, sizeof(double));
    double* alphas = (double*)calloc(hist_cap + 1, sizeof(double));
    double j = obj_eval(o, y, grad);
    const double g0 = vec_norm(grad, n);
    const double min_hy = obj_min_spacing(o);
    op_t op = {o, 1, gamma};
    for (int it = 0; it < cfg->max_iters; ++it) {
        mport_iter_record rec = {it, 0, j, o->last_distance, o->last_regularizer, vec_norm(grad, n), 0.0};
        if (rec.grad_norm <= cfg->tol_grad * g0) {
            push_rec(tr, cap, nt, &rec);
            break;
        }
        /* direction, optimizer.cpp:285-312 */
        memcpy(q, grad, sizeof(double) * n);
        for (int k = hn; k-- > 0;) {
            alphas[k] = hrho[k] * vec_dot(hs[k], q, n);
            for (int64_t i = 0; i < n; ++i) q[i] -= alphas[k] * hy[k][i];
        }
        int iters, brk;
        double relres;
        cg_solve(&op, q, n, cfg->h0_max_iters, cfg->h0_rel_tol, r, &iters, &relres, &brk);
        for (int k = 0; k < hn; ++k) {
            const double beta = hrho[k] * vec_dot(hy[k], r, n);
            for (int64_t i = 0; i < n; ++i) r[i] += (alphas[k] - beta) * hs[k][i];
        }
        for (int64_t i = 0; i < n; ++i) dir[i] = -r[i];
        rec.cg_iters = iters;
        const double gdotd = vec_dot(grad, dir, n);
        const double dinf = vec_inf_norm(dir, n);
        double eta0 = 1.0;
        if (dinf > 0.0) {
            const double qq = min_hy / dinf;
            eta0 = qq < 1.0 ? qq : 1.0;
        }
        double eta = 0.0;
        if (!armijo(o, y, dir, yt, n, j, gdotd, cfg, eta0, &eta)) {
            *lsf = 1;
            push_rec(tr, cap, nt, &rec);
            break;
        }
        rec.step = eta;
        const double j_prev = j;
        double* s = (double*)calloc(n, sizeof(double));
        double step_inf = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            s[i] = eta * dir[i];
            y[i] += s[i];
            const double as = fabs(s[i]);
            step_inf = step_inf < as ? as : step_inf;
        }
        j = obj_eval(o, y, gnew);
        double* yv = (double*)calloc(n, sizeof(double));
        for (int64_t i = 0; i < n; ++i) yv[i] = gnew[i] - grad[i];
        const double sy = vec_dot(s, yv, n);
        if (sy > 1e-10 * vec_norm(s, n) * vec_norm(yv, n)) {
            hs[hn] = s;
            hy[hn] = yv;
            hrho[hn] = 1.0 / sy;
            ++hn;
            while (hn > hist_cap) { /* pop_front */
                free(hs[0]);
                free(hy[0]);
                memmove(hs, hs + 1, sizeof(double*) * (hn - 1));
                memmove(hy, hy + 1, sizeof(double*) * (hn - 1));
                memmove(hrho, hrho + 1, sizeof(double) * (hn - 1));
                --hn;
            }
        } else {
            free(s);
            free(yv);
        }
        memcpy(grad, gnew, sizeof(double) * n);
        push_rec(tr, cap, nt, &rec);
        if (should_stop(cfg, g0, min_hy, j_prev, j, vec_norm(grad, n), step_inf)) break;
    }
    for (int k = 0; k < hn; ++k) { free(hs[k]); free(hy[k]); }
    free(hs); free(hy); free(hrho); free(grad); free(gnew); free(dir); free(yt); free(q); free(r); free(alphas);
}

/* ------------------------------------------------------------ multilevel */
/* multilevel.cpp:39-49 */
static int deformation_grid_for(const grid_t* img, int64_t ratio, grid_t* out) {
    if (ratio < 1) return fail(E_INVALID, "deformation_grid_for: ratio must be >= 1");
    int64_t pts[3];
    for (int a = 0; a < 3; ++a) {
        const int64_t v = (img->m[a] + ratio - 1) / ratio + 1;
        pts[a] = v > 2 ? v : 2;
    }
    return make_deform_grid(img, pts, out);
}

/* multilevel.cpp:51-76 */
static double nodal_interpolate(const double* comp, const grid_t* g, const double p[3]) {
    int64_t b[3];
    double w[3];
    for (int a = 0; a < 3; ++a) {
        const int64_t ma = g->m[a];
        double s = p[a] / g->h[a];
        const double hi = (double)(ma - 1);
        s = (s < 0.0) ? 0.0 : ((hi < s) ? hi : s);
        int64_t base = (int64_t)floor(s);
        if (base < 0) base = 0;
        if (base > ma - 2) base = ma - 2;
        b[a] = base;
        w[a] = s - (double)base;
    }
    double v = 0.0;
    for (int c = 0; c < 2; ++c)
        for (int bb = 0; bb < 2; ++bb)
            for (int aa = 0; aa < 2; ++aa) {
                const double weight = (aa ? w[0] : 1.0 - w[0]) * (bb ? w[1] : 1.0 - w[1]) * (c ? w[2] : 1.0 - w[2]);
                v += weight * comp[g_linear(g, b[0] + aa, b[1] + bb, b[2] + c)];
            }
    return v;
}

/* multilevel.cpp:78-115 */
static int prolong(const double* yc, const grid_t* c, const grid_t* f, double* out) {
    int rc = g_validate(c);
    if (rc || (rc = g_validate(f))) return rc;
    for (int a = 0; a < 3; ++a) {
        const double tol = c->h[a] > f->h[a] ? c->h[a] : f->h[a];
        if (fabs(g_extent(c, a) - g_extent(f, a)) > tol) return fail(E_INVALID, "prolong: grid extents differ");
    }
    const int64_t nc = g_count(c), nf = g_count(f);
    double* u = (double*)malloc(sizeof(double) * 3 * nc);
    for (int64_t i = 0; i < nc; ++i) {
        double x[3];
        g_point(c, i, x);
        for (int d = 0; d < 3; ++d) u[d * nc + i] = yc[d * nc + i] - x[d];
    }
    for (int64_t i = 0; i < nf; ++i) {
        double x[3];
        g_point(f, i, x);
        for (int d = 0; d < 3; ++d) out[d * nf + i] = x[d] + nodal_interpolate(u + d * nc, c, x);
    }
    free(u);
    return OK;
}

/* ------------------------------------------------------------- synthetic */
/* std::mt19937_64 (the reference's RNG, synthetic.cpp:69,115) */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;
static void mt_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt_next(mt64_t* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* libstdc++ generate_canonical<double,53> + uniform_real_distribution: c*(b-a)+a */
static double uniform_real(mt64_t* s, double a, double b) {
    double c = (double)mt_next(s) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return (c * (b - a)) + a;
}
/* libstdc++ uniform_int_distribution (Lemire downscaling for a 64-bit engine) */
static int uniform_int(mt64_t* s, int a, int b) {
    const uint64_t range = (uint64_t)((int64_t)b - (int64_t)a) + 1;
    unsigned __int128 prod = (unsigned __int128)mt_next(s) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t thr = (0 - range) % range;
        while (low < thr) {
            prod = (unsigned __int128)mt_next(s) * range;
            low = (uint64_t)prod;
        }
    }
    return a + (int)(uint64_t)(prod >> 64);
}

static double soft_step(double x, double width) { return 1.0 / (1.0 + exp(-x / width)); }
#define PI 3.141592653589793

/* synthetic.cpp:15-63 */
int mport_make_phantom(const int64_t* m, const double* h, double* out) {
    const grid_t g = image_grid(m, h);
    int rc = g_validate(&g);
    if (rc) return rc;
    const double e[3] = {g_extent(&g, 0), g_extent(&g, 1), g_extent(&g, 2)};
    double scale = e[0];
    if (e[1] < scale) scale = e[1];
    if (e[2] < scale) scale = e[2];
    const double edge = 0.015 * scale;
    static const double sc[5][3] = {{0.35, 0.4, 0.45}, {0.68, 0.62, 0.40}, {0.55, 0.30, 0.68},
                                    {0.30, 0.70, 0.62}, {0.72, 0.35, 0.70}};
    static const double sr[5] = {0.22, 0.14, 0.10, 0.08, 0.06};
    static const double sw[5] = {1.0, -0.7, 0.8, 0.6, -0.5};
    const int64_t n = g_count(&g);
    for (int64_t i = 0; i < n; ++i) {
        double p[3];
        g_point(&g, i, p);
        double val = 0.1 * (p[0] / e[0]) * (p[1] / e[1]);
        for (int s = 0; s < 5; ++s) {
            double d2 = 0.0;
            for (int a = 0; a < 3; ++a) {
                const double diff = p[a] - sc[s][a] * e[a];
                d2 += diff * diff;
            }
            val += sw[s] * soft_step(sr[s] * scale - sqrt(d2), edge);
        }
        const double plane = (p[0] / e[0] + p[1] / e[1] + p[2] / e[2]) / 3.0 - 0.55;
        val += 0.4 * soft_step(-fabs(plane) + 0.04, 0.01);
        const double tx = 2.0 * PI * p[0] / e[0];
        const double ty = 2.0 * PI * p[1] / e[1];
        const double tz = 2.0 * PI * p[2] / e[2];
        val += 0.12 * sin(3.0 * tx + 0.8 * sin(2.0 * ty)) * cos(2.0 * ty + 0.6 * sin(3.0 * tz)) +
               0.08 * cos(4.0 * tz + 0.7 * sin(2.0 * tx)) * sin(3.0 * ty + 0.5 * cos(2.0 * tx));
        out[i] = val;
    }
    return OK;
}

/* synthetic.cpp:65-90 */
int mport_make_random_volume(const int64_t* m, const double* h, uint64_t seed, int passes, double* out) {
    const grid_t g = image_grid(m, h);
    int rc = g_validate(&g);
    if (rc) return rc;
    const int64_t n = g_count(&g);
    mt64_t rng;
    mt_seed(&rng, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = uniform_real(&rng, 0.0, 1.0);
    double* tmp = (double*)malloc(sizeof(double) * n);
    for (int pass = 0; pass < passes; ++pass) {
        for (int64_t i = 0; i < n; ++i) {
            double s = out[i];
            for (int d = 0; d < 7; ++d) {
                if (d == CENTER) continue;
                s += out[g_neighbor(&g, i, d)];
            }
            tmp[i] = s / 7.0;
        }
        memcpy(out, tmp, sizeof(double) * n);
    }
    free(tmp);
    return OK;
}

typedef struct {
    double extent[3];
    double amp[3][3];
    int freq[3][3];
    double phase[3][3];
} warp_t;

/* synthetic.cpp:110-143 */
static void make_sinusoid_warp(const double* extent, double max_amp, uint64_t seed, warp_t* w) {
    for (int a = 0; a < 3; ++a) w->extent[a] = extent[a];
    mt64_t rng;
    mt_seed(&rng, seed);
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) {
            w->amp[t][d] = uniform_real(&rng, -1.0, 1.0);
            w->freq[t][d] = uniform_int(&rng, 1, 2);
            w->phase[t][d] = uniform_real(&rng, -0.5, 0.5);
        }
    double bound = 0.0;
    for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int t = 0; t < 3; ++t) s += fabs(w->amp[t][d]);
        bound = bound < s ? s : bound;
    }
    const double scale = bound > 0.0 ? max_amp / (bound * sqrt(3.0)) : 0.0;
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) w->amp[t][d] *= scale;
}

/* synthetic.cpp:92-108 */
static void warp_displacement(const warp_t* w, const double p[3], double u[3]) {
    u[0] = u[1] = u[2] = 0.0;
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) {
            double v = w->amp[t][d];
            for (int a = 0; a < 3; ++a) {
                const double x = p[a] / w->extent[a];
                v *= sin(PI * w->freq[t][a] * x + w->phase[t][a] * x * (1.0 - x));
            }
            u[d] += v;
        }
}

int mport_sinusoid_terms(const double* extent, double max_amp, uint64_t seed, double* amp, int* freq,
                         double* phase) {
    warp_t w;
    make_sinusoid_warp(extent, max_amp, seed, &w);
    for (int t = 0; t < 3; ++t)
        for (int d = 0; d < 3; ++d) {
            amp[t * 3 + d] = w.amp[t][d];
            freq[t * 3 + d] = w.freq[t][d];
            phase[t * 3 + d] = w.phase[t][d];
        }
    return OK;
}

/* synthetic.cpp:145-159 */
int mport_warp_sinusoid(const double* vol, const int64_t* m, const double* h, double max_amp, uint64_t seed,
                        double* out) {
    const grid_t g = image_grid(m, h);
    int rc = g_validate(&g);
    if (rc) return rc;
    const double ext[3] = {g_extent(&g, 0), g_extent(&g, 1), g_extent(&g, 2)};
    warp_t w;
    make_sinusoid_warp(ext, max_amp, seed, &w);
    const int64_t n = g_count(&g);
    for (int64_t i = 0; i < n; ++i) {
        double p[3], u[3], gr[3];
        g_point(&g, i, p);
        warp_displacement(&w, p, u);
        for (int d = 0; d < 3; ++d) p[d] += u[d];
        interpolate(vol, &g, p, &out[i], gr);
    }
    return OK;
}

/* synthetic.cpp:161-175 */
int mport_warp_field(const int64_t* m, const double* h, double max_amp, uint64_t seed, const int64_t* my,
                     double* out) {
    const grid_t img = image_grid(m, h);
    int rc = g_validate(&img);
    if (rc) return rc;
    const double ext[3] = {g_extent(&img, 0), g_extent(&img, 1), g_extent(&img, 2)};
    warp_t w;
    make_sinusoid_warp(ext, max_amp, seed, &w);
    grid_t dg;
    if ((rc = make_deform_grid(&img, my, &dg))) return rc;
    const int64_t n = g_count(&dg);
    for (int64_t i = 0; i < n; ++i) {
        double p[3], u[3];
        g_point(&dg, i, p);
        warp_displacement(&w, p, u);
        for (int d = 0; d < 3; ++d) out[d * n + i] = p[d] + u[d];
    }
    return OK;
}

/* ------------------------------------------------------- C entry points */
int mport_make_deform_grid(const int64_t* m, const double* h, const int64_t* my, double* hy) {
    const grid_t img = image_grid(m, h);
    int rc = g_validate(&img);
    if (rc) return rc;
    grid_t dg;
    if ((rc = make_deform_grid(&img, my, &dg))) return rc;
    for (int a = 0; a < 3; ++a) hy[a] = dg.h[a];
    return OK;
}

int mport_deformation_grid_for(const int64_t* m, const double* h, int64_t ratio, int64_t* my, double* hy) {
    const grid_t img = image_grid(m, h);
    int rc = g_validate(&img);
    if (rc) return rc;
    grid_t dg;
    if ((rc = deformation_grid_for(&img, ratio, &dg))) return rc;
    for (int a = 0; a < 3; ++a) {
        my[a] = dg.m[a];
        hy[a] = dg.h[a];
    }
    return OK;
}

int mport_transfer_plan(const int64_t* ms, const double* hs, const int64_t* mt, const double* ht, int64_t* base,
                        double* rem) {
    const grid_t s = nodal_grid(ms, hs), t = image_grid(mt, ht);
    plan_t p;
    int rc = make_plan(&s, &t, &p);
    if (rc) return rc;
    int64_t o = 0;
    for (int a = 0; a < 3; ++a)
        for (int64_t k = 0; k < mt[a]; ++k, ++o) {
            base[o] = p.base[a][k];
            rem[o] = p.rem[a][k];
        }
    plan_free(&p);
    return OK;
}

int mport_transfer_apply(const int64_t* ms, const double* hs, const int64_t* mt, const double* ht, const double* y,
                         double* out) {
    const grid_t s = nodal_grid(ms, hs), t = image_grid(mt, ht);
    plan_t p;
    int rc = make_plan(&s, &t, &p);
    if (rc) return rc;
    transfer_apply(&p, y, out);
    plan_free(&p);
    return OK;
}

int mport_transfer_apply_transpose(const int64_t* ms, const double* hs, const int64_t* mt, const double* ht,
                                   const double* w, double* out) {
    const grid_t s = nodal_grid(ms, hs), t = image_grid(mt, ht);
    plan_t p;
    int rc = make_plan(&s, &t, &p);
    if (rc) return rc;
    transfer_apply_transpose(&p, w, out);
    plan_free(&p);
    return OK;
}

int mport_interpolate(const double* t, const int64_t* m, const double* h, const double* p, double* value,
                      double* grad) {
    const grid_t g = image_grid(m, h);
    interpolate(t, &g, p, value, grad);
    return OK;
}

int mport_sample_deformed(const double* t, const int64_t* m, const double* h, const double* points, int64_t n,
                          double* values, double* partials) {
    const grid_t g = image_grid(m, h);
    int rc = g_validate(&g);
    if (rc) return rc;
    sample_deformed(t, &g, points, n, values, partials);
    return OK;
}

int mport_downsample(const double* v, const int64_t* m, const double* h, double* out, int64_t* mo, double* ho) {
    const grid_t g = image_grid(m, h);
    grid_t c;
    int rc = downsample(v, &g, out, &c);
    if (rc) return rc;
    for (int a = 0; a < 3; ++a) {
        mo[a] = c.m[a];
        ho[a] = c.h[a];
    }
    return OK;
}

typedef struct {
    ngf_t* ngf;
} ngf_handle;

void* mport_ngf_create(const double* ref, const int64_t* m, const double* h, double tau, double rho) {
    const grid_t g = image_grid(m, h);
    int rc = g_validate(&g);
    if (rc) return NULL;
    ngf_t* c = ngf_new(ref, &g, tau, rho, &rc);
    return c;
}
void mport_ngf_destroy(void* p) { ngf_free((ngf_t*)p); }
int mport_ngf_populate(void* p, const double* tpl, const double* points) {
    return ngf_populate((ngf_t*)p, tpl, points);
}
int mport_ngf_workspace(void* p, double* values, double* partials, double* tpl_grads, double* residual,
                        double* inv1, double* inv2, double* ref_grads, double* ref_norms) {
    const ngf_t* c = (const ngf_t*)p;
    const int64_t n = g_count(&c->g);
    for (int64_t i = 0; i < n; ++i) {
        if (values) values[i] = c->values[i];
        if (partials)
            for (int a = 0; a < 3; ++a) partials[a * n + i] = c->partials[a * n + i];
        if (tpl_grads)
            for (int k = 0; k < 6; ++k) tpl_grads[k * n + i] = c->tpl_grads[6 * i + k];
        if (ref_grads)
            for (int k = 0; k < 6; ++k) ref_grads[k * n + i] = c->ref_grads[6 * i + k];
        if (ref_norms) ref_norms[i] = c->ref_norms[i];
        if (residual) residual[i] = c->residual[i];
        if (inv1) inv1[i] = c->inv1[i];
        if (inv2) inv2[i] = c->inv2[i];
    }
    return OK;
}
int mport_ngf_value(void* p, double* out) {
    *out = ngf_value((const ngf_t*)p);
    return OK;
}
int mport_ngf_gradient(void* p, double* out) {
    ngf_gradient((const ngf_t*)p, out);
    return OK;
}
int mport_ngf_hessian_vec(void* p, const double* v, double* out) {
    return ngf_hessian_vec((const ngf_t*)p, v, out);
}
int mport_ngf_rho(void* p, int64_t i, int k, double* out) {
    const ngf_t* c = (const ngf_t*)p;
    double hh[3];
    hhat(&c->g, hh);
    *out = rho_hat(c, i, k, hh);
    return OK;
}

int mport_laplacian_apply(const double* u, const int64_t* m, const double* h, double* out) {
    const grid_t g = nodal_grid(m, h);
    const int64_t n = g_count(&g);
    for (int64_t i = 0; i < n; ++i) out[i] = laplacian(u, &g, i);
    return OK;
}
int mport_curvature_value(const double* u, const int64_t* m, const double* h, double* out) {
    const grid_t g = nodal_grid(m, h);
    *out = curvature_value(u, &g);
    return OK;
}
int mport_curvature_gradient(const double* u, const int64_t* m, const double* h, double* out) {
    const grid_t g = nodal_grid(m, h);
    double* scratch = (double*)calloc(g_count(&g), sizeof(double));
    biharmonic(u, &g, scratch, out);
    free(scratch);
    return OK;
}
int mport_curvature_hessian_vec(const double* u, const int64_t* m, const double* h, double* out) {
    return mport_curvature_gradient(u, m, h, out);
}

void* mport_objective_create(const double* ref, const double* tpl, const int64_t* m, const double* h,
                             const int64_t* my, double tau, double rho, double alpha) {
    const grid_t img = image_grid(m, h);
    int rc = g_validate(&img);
    if (rc) return NULL;
    grid_t dg;
    if ((rc = make_deform_grid(&img, my, &dg))) return NULL;
    return obj_new(ref, tpl, &img, &dg, tau, rho, alpha, &rc);
}
void mport_objective_destroy(void* p) { obj_free((obj_t*)p); }
int64_t mport_objective_dof(void* p) { return obj_dof((obj_t*)p); }
int mport_objective_identity(void* p, double* out) {
    obj_t* o = (obj_t*)p;
    memcpy(out, o->xid, sizeof(double) * obj_dof(o));
    return OK;
}
int mport_objective_eval(void* p, const double* y, double* grad, double* j, double* dist, double* reg) {
    obj_t* o = (obj_t*)p;
    *j = obj_eval(o, y, grad);
    *dist = o->last_distance;
    *reg = o->last_regularizer;
    return OK;
}
int mport_objective_gn_hessian_vec(void* p, const double* v, double* q) {
    obj_gn_hv((obj_t*)p, v, q);
    return OK;
}
int mport_objective_seed_hessian_vec(void* p, const double* v, double gamma, double* q) {
    obj_seed_hv((obj_t*)p, v, gamma, q);
    return OK;
}
int mport_cg_solve(void* p, int seed, double gamma, const double* b, int max_iters, double rel_tol, double* x,
                   int* iters, double* relres, int* breakdown) {
    obj_t* o = (obj_t*)p;
    op_t op = {o, seed, gamma};
    cg_solve(&op, b, obj_dof(o), max_iters, rel_tol, x, iters, relres, breakdown);
    return OK;
}
int mport_minimize(void* p, int method, const double* y0, const mport_opt_config* cfg, double* y_out,
                   mport_iter_record* trace, int cap, int* ntrace, int* ls_failed) {
    obj_t* o = (obj_t*)p;
    if (method == 1) gauss_newton(o, y0, cfg, y_out, trace, cap, ntrace, ls_failed);
    else lbfgs(o, y0, cfg, y_out, trace, cap, ntrace, ls_failed);
    return OK;
}
int mport_prolong(const double* yc, const int64_t* mc, const double* hc, const int64_t* mf, const double* hf,
                  double* out) {
    const grid_t c = nodal_grid(mc, hc), f = nodal_grid(mf, hf);
    return prolong(yc, &c, &f, out);
}

/* multilevel.cpp:9-37 + 117-145 */
int mport_register_multilevel(const double* ref, const double* tpl, const int64_t* m, const double* h, int levels,
                              int64_t ratio, double tau, double rho, double alpha, int method,
                              const mport_opt_config* cfg, double* y_out, mport_iter_record* trace, int cap,
                              int* level_iters, int* ls_failed) {
    if (levels < 1) return fail(E_INVALID, "build_pyramid: levels must be >= 1");
    const grid_t g0 = image_grid(m, h);
    int rc = g_validate(&g0);
    if (rc) return rc;
    for (int a = 0; a < 3; ++a) {
        int64_t mm = m[a];
        for (int l = 1; l < levels; ++l) {
            if (mm < 2) return fail(E_INVALID, "build_pyramid: too many levels for this size");
            mm = (mm + 1) / 2;
        }
        if (mm < 2) return fail(E_INVALID, "build_pyramid: too many levels for this size");
    }
    double** R = (double**)calloc(levels, sizeof(double*));
    double** T = (double**)calloc(levels, sizeof(double*));
    grid_t* G = (grid_t*)calloc(levels, sizeof(grid_t));
    const int64_t n0 = g_count(&g0);
    R[0] = (double*)malloc(sizeof(double) * n0);
    T[0] = (double*)malloc(sizeof(double) * n0);
    memcpy(R[0], ref, sizeof(double) * n0);
    memcpy(T[0], tpl, sizeof(double) * n0);
    G[0] = g0;
    for (int l = 1; l < levels; ++l) {
        downsample(R[l - 1], &G[l - 1], NULL, &G[l]);
        R[l] = (double*)malloc(sizeof(double) * g_count(&G[l]));
        T[l] = (double*)malloc(sizeof(double) * g_count(&G[l]));
        downsample(R[l - 1], &G[l - 1], R[l], &G[l]);
        downsample(T[l - 1], &G[l - 1], T[l], &G[l]);
    }
    double* y = NULL;
    grid_t prev;
    int have_prev = 0, off = 0, li = 0;
    for (int l = levels - 1; l >= 0; --l, ++li) {
        grid_t dg;
        if ((rc = deformation_grid_for(&G[l], ratio, &dg))) break;
        obj_t* o = obj_new(R[l], T[l], &G[l], &dg, tau, rho, alpha, &rc);
        if (!o) break;
        const int64_t nd = obj_dof(o);
        double* y0 = (double*)malloc(sizeof(double) * nd);
        if (have_prev) prolong(y, &prev, &dg, y0);
        else memcpy(y0, o->xid, sizeof(double) * nd);
        free(y);
        y = (double*)malloc(sizeof(double) * nd);
        int nt = 0, lsf = 0;
        mport_iter_record* tr = trace ? trace + (off < cap ? off : cap) : NULL;
        const int room = off < cap ? cap - off : 0;
        if (method == 1) gauss_newton(o, y0, cfg, y, tr, room, &nt, &lsf);
        else lbfgs(o, y0, cfg, y, tr, room, &nt, &lsf);
        level_iters[li] = nt;
        ls_failed[li] = lsf;
        off += nt;
        free(y0);
        obj_free(o);
        prev = dg;
        have_prev = 1;
    }
    if (!rc && y) memcpy(y_out, y, sizeof(double) * 3 * g_count(&prev));
    free(y);
    for (int l = 0; l < levels; ++l) { free(R[l]); free(T[l]); }
    free(R); free(T); free(G);
    return rc;
}
