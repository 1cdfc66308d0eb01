/* CPU restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.
 * See wmc_oracle.h.  Every function cites the reference code it restates
 * (paths relative to /root/reference/proj).  It is a straight, scalar
 * restatement: a CSR operator over all interior rows, the LTS recursion in
 * deviation form over every row, a check for blow-up after every step.
 */
#include "wmc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- RNG: include/wavemc/rng.hpp:14-19, src/rng.cpp:10-32 ---- */

uint64_t wmc_oracle_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static uint64_t stream_key(uint64_t seed, uint32_t level, uint64_t index) {
    uint64_t k = wmc_oracle_mix64(seed);
    k = wmc_oracle_mix64(k ^ (0xa511e9b3cc1f25d1ULL + (uint64_t)level));
    k = wmc_oracle_mix64(k ^ (0x63d1c71ad3e29f0bULL + index));
    return k;
}

void wmc_oracle_stream_words(uint64_t seed, uint32_t level, uint64_t index, int count, uint64_t* out) {
    const uint64_t key = stream_key(seed, level, index);
    for (int c = 0; c < count; ++c) out[c] = wmc_oracle_mix64(key + (uint64_t)c * 0x9e3779b97f4a7c15ULL);
}

/* next_uniform(lo, hi) = lo + (hi - lo) * ((word >> 11) * 2^-53), one word per cell */
void wmc_oracle_draw_cells(uint64_t seed, uint32_t level, uint64_t index, int n_cells, double lo, double hi,
                           double* out) {
    const uint64_t key = stream_key(seed, level, index);
    for (int c = 0; c < n_cells; ++c) {
        const uint64_t w = wmc_oracle_mix64(key + (uint64_t)c * 0x9e3779b97f4a7c15ULL);
        out[c] = lo + (hi - lo) * ((double)(w >> 11) * 0x1.0p-53);
    }
}

/* Log-normal KL on the cell grid -- not in the reference (its only KL field is
 * 1D with U(-1,1) weights, src/rng.cpp:42-51); the same definition as the
 * device draw: words 2i, 2i+1 -> u1, u2 (next_unit), r = sqrt(-2 log(1-u1)),
 * xi_2i = r cos(2 pi u2), xi_2i+1 = r sin(2 pi u2), c_k = exp(sum T[k][m] xi_m). */
void wmc_oracle_draw_kl(uint64_t seed, uint32_t level, uint64_t index, const double* table, int n_cells, int modes,
                        double* out) {
    const uint64_t key = stream_key(seed, level, index);
    double xi[128];
    const double two_pi = 6.283185307179586;
    for (int i = 0; 2 * i < modes && 2 * i < 128; ++i) {
        const uint64_t w1 = wmc_oracle_mix64(key + (uint64_t)(2 * i) * 0x9e3779b97f4a7c15ULL);
        const uint64_t w2 = wmc_oracle_mix64(key + (uint64_t)(2 * i + 1) * 0x9e3779b97f4a7c15ULL);
        const double u1 = (double)(w1 >> 11) * 0x1.0p-53, u2 = (double)(w2 >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(1.0 - u1)), th = two_pi * u2;
        xi[2 * i] = r * cos(th);
        if (2 * i + 1 < modes) xi[2 * i + 1] = r * sin(th);
    }
    for (int k = 0; k < n_cells; ++k) {
        double g = 0.0;
        for (int m = 0; m < modes; ++m) g += table[k * modes + m] * xi[m];
        out[k] = exp(g);
    }
}

/* ---- Chebyshev constants: src/integrators.cpp:34-66 ---- */

int wmc_oracle_chebyshev(int p, double nu, double* delta, double* omega, double* beta_int, double* beta_half) {
    if (p < 1 || nu < 0.0 || nu > 1.0) return 2;
    const double d = 1.0 + nu / ((double)p * p);
    double* t = (double*)malloc(sizeof(double) * (size_t)(p + 2));
    t[0] = 1.0;
    t[1] = d;
    for (int k = 2; k <= p; ++k) t[k] = 2.0 * d * t[k - 1] - t[k - 2];
    double u_prev = 1.0, u = 2.0 * d;
    for (int k = 2; k <= p - 1; ++k) {
        const double next = 2.0 * d * u - u_prev;
        u_prev = u;
        u = next;
    }
    const double u_pm1 = (p == 1) ? 1.0 : u;
    *delta = d;
    *omega = 2.0 * p * u_pm1 / t[p];
    for (int k = 1; k <= p - 1; ++k) {
        beta_int[k - 1] = t[k - 1] / t[k + 1];
        beta_half[k - 1] = t[k] / t[k + 1];
    }
    free(t);
    return 0;
}

/* ---- operator: src/fem.cpp:91-126 (assemble), :42-63 (make_operator,
 *      normalize), include/wavemc/sparse.hpp:17-77 (CSR, masked columns) ---- */

typedef struct {
    int n;
    int* rp;
    int* ci;
    double* va;
} csr;

typedef struct {
    int row, col;
    double v;
} trip;

static int trip_cmp(const void* a, const void* b) {
    const trip* x = (const trip*)a;
    const trip* y = (const trip*)b;
    if (x->row != y->row) return x->row < y->row ? -1 : 1;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return 0;
}

/* from_triplets: sort by (row, col), sum duplicates (sparse.hpp:17-40) */
static csr csr_from_triplets(int n, trip* t, long nt) {
    qsort(t, (size_t)nt, sizeof(trip), trip_cmp);
    csr m;
    m.n = n;
    m.rp = (int*)calloc((size_t)n + 1, sizeof(int));
    m.ci = (int*)malloc(sizeof(int) * (size_t)(nt ? nt : 1));
    m.va = (double*)malloc(sizeof(double) * (size_t)(nt ? nt : 1));
    long k = 0;
    for (long i = 0; i < nt;) {
        const int r = t[i].row, c = t[i].col;
        double v = 0.0;
        while (i < nt && t[i].row == r && t[i].col == c) v += t[i++].v;
        m.ci[k] = c;
        m.va[k] = v;
        ++k;
        m.rp[r + 1]++;
    }
    for (int r = 0; r < n; ++r) m.rp[r + 1] += m.rp[r];
    return m;
}

static void csr_free(csr* m) {
    free(m->rp);
    free(m->ci);
    free(m->va);
}

/* multiply: y_r = sum_k va[k] x[ci[k]] in column order (sparse.hpp:46-52) */
static void csr_mul(const csr* m, const double* x, double* y) {
    for (int r = 0; r < m->n; ++r) {
        double acc = 0.0;
        for (int k = m->rp[r]; k < m->rp[r + 1]; ++k) acc += m->va[k] * x[m->ci[k]];
        y[r] = acc;
    }
}

/* masked_columns (sparse.hpp:61-77) */
static csr csr_mask(const csr* a, const unsigned char* keep, int want) {
    csr m;
    m.n = a->n;
    m.rp = (int*)calloc((size_t)a->n + 1, sizeof(int));
    long nnz = a->rp[a->n];
    m.ci = (int*)malloc(sizeof(int) * (size_t)(nnz ? nnz : 1));
    m.va = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    long k2 = 0;
    for (int r = 0; r < a->n; ++r) {
        for (int k = a->rp[r]; k < a->rp[r + 1]; ++k)
            if ((keep[a->ci[k]] != 0) == (want != 0)) {
                m.ci[k2] = a->ci[k];
                m.va[k2] = a->va[k];
                ++k2;
            }
        m.rp[r + 1] = (int)k2;
    }
    return m;
}

typedef struct {
    int n;                /* interior vertices */
    int* dof_vertex;
    double* mass;         /* lumped mass per dof */
    unsigned char* sel;   /* selector per dof */
    unsigned char* vt;    /* nested tiers: largest flag (capped at tiers) of the dof's triangles */
    csr a, a_fine, a_coarse;
} oper;

/* cell k = iy * cells_x + ix, ix = floor((x - x0) / (x1 - x0) * cells_x) over the domain box */
static int cell_of(const wmc_oracle_problem* pb, double x, double y) {
    const int unit = pb->domain[0] == 0.0 && pb->domain[1] == 0.0 && pb->domain[2] == 0.0 && pb->domain[3] == 0.0;
    const double x0 = unit ? 0.0 : pb->domain[0], x1 = unit ? 1.0 : pb->domain[1];
    const double y0 = unit ? 0.0 : pb->domain[2], y1 = unit ? 1.0 : pb->domain[3];
    int ix = (int)floor((x - x0) / (x1 - x0) * pb->cells_x), iy = (int)floor((y - y0) / (y1 - y0) * pb->cells_y);
    if (ix < 0) ix = 0;
    if (ix > pb->cells_x - 1) ix = pb->cells_x - 1;
    if (iy < 0) iy = 0;
    if (iy > pb->cells_y - 1) iy = pb->cells_y - 1;
    return iy * pb->cells_x + ix;
}

static double tri_area(const wmc_oracle_mesh* m, int t) {
    const double* a = m->xy + 2 * m->tri[3 * t];
    const double* b = m->xy + 2 * m->tri[3 * t + 1];
    const double* c = m->xy + 2 * m->tri[3 * t + 2];
    return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
}

static void tri_centroid(const wmc_oracle_mesh* m, int t, double* cx, double* cy) {
    const double* a = m->xy + 2 * m->tri[3 * t];
    const double* b = m->xy + 2 * m->tri[3 * t + 1];
    const double* c = m->xy + 2 * m->tri[3 * t + 2];
    *cx = (a[0] + b[0] + c[0]) / 3.0;
    *cy = (a[1] + b[1] + c[1]) / 3.0;
}

/* assemble with speed2 = cells[cell(centroid)], Dirichlet by keeping interior rows/cols */
static int build_operator(const wmc_oracle_mesh* m, const wmc_oracle_problem* pb, const double* cells, oper* op) {
    const int nv = m->n_vertices, nt = m->n_triangles;
    double* vmass = (double*)calloc((size_t)nv, sizeof(double));
    int* dof = (int*)malloc(sizeof(int) * (size_t)nv);
    int n = 0;
    for (int v = 0; v < nv; ++v) dof[v] = m->boundary[v] ? -1 : n++;
    trip* t = (trip*)malloc(sizeof(trip) * (size_t)(9 * (long)nt + 1));
    long ntrip = 0;
    for (int e = 0; e < nt; ++e) {
        const int* tv = m->tri + 3 * e;
        const double* p0 = m->xy + 2 * tv[0];
        const double* p1 = m->xy + 2 * tv[1];
        const double* p2 = m->xy + 2 * tv[2];
        const double area = tri_area(m, e);
        if (!(area > 0.0)) {
            free(vmass);
            free(dof);
            free(t);
            return 3;
        }
        double cx, cy;
        tri_centroid(m, e, &cx, &cy);
        const double c2 = cells[cell_of(pb, cx, cy)];
        const double gx[3] = {(p1[1] - p2[1]) / (2.0 * area), (p2[1] - p0[1]) / (2.0 * area),
                              (p0[1] - p1[1]) / (2.0 * area)};
        const double gy[3] = {(p2[0] - p1[0]) / (2.0 * area), (p0[0] - p2[0]) / (2.0 * area),
                              (p1[0] - p0[0]) / (2.0 * area)};
        for (int i = 0; i < 3; ++i) {
            vmass[tv[i]] += area / 3.0;
            for (int j = 0; j < 3; ++j) {
                if (dof[tv[i]] < 0 || dof[tv[j]] < 0) continue;
                t[ntrip].row = dof[tv[i]];
                t[ntrip].col = dof[tv[j]];
                t[ntrip].v = c2 * area * (gx[i] * gx[j] + gy[i] * gy[j]);
                ++ntrip;
            }
        }
    }
    op->n = n;
    op->dof_vertex = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
    op->mass = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    op->sel = (unsigned char*)calloc((size_t)(n ? n : 1), 1);
    op->vt = (unsigned char*)calloc((size_t)(n ? n : 1), 1);
    for (int v = 0; v < nv; ++v)
        if (dof[v] >= 0) {
            op->dof_vertex[dof[v]] = v;
            op->mass[dof[v]] = vmass[v];
        }
    const int tiers = pb->tiers > 1 ? pb->tiers : 1;
    for (int e = 0; e < nt; ++e)
        if (m->fine[e])
            for (int i = 0; i < 3; ++i) {
                const int d = dof[m->tri[3 * e + i]];
                if (d < 0) continue;
                const int f = m->fine[e] < tiers ? m->fine[e] : tiers;
                op->sel[d] = 1;
                if (f > op->vt[d]) op->vt[d] = (unsigned char)f;
            }
    csr k = csr_from_triplets(n, t, ntrip);
    /* normalize: A_ij = K_ij / sqrt(M_i M_j) */
    for (int r = 0; r < n; ++r)
        for (int q = k.rp[r]; q < k.rp[r + 1]; ++q) k.va[q] = k.va[q] / sqrt(op->mass[r] * op->mass[k.ci[q]]);
    op->a = k;
    op->a_fine = csr_mask(&op->a, op->sel, 1);
    op->a_coarse = csr_mask(&op->a, op->sel, 0);
    free(vmass);
    free(dof);
    free(t);
    return 0;
}

static void oper_free(oper* op) {
    free(op->dof_vertex);
    free(op->mass);
    free(op->sel);
    free(op->vt);
    csr_free(&op->a);
    csr_free(&op->a_fine);
    csr_free(&op->a_coarse);
}

/* lumped L2 projection, edge-midpoint rule, z0 = sqrt(M) coef (fem.cpp:223-255) */
static void project_z0(const wmc_oracle_mesh* m, const wmc_oracle_problem* pb, const oper* op, double* z0) {
    const int nv = m->n_vertices;
    double* load = (double*)calloc((size_t)nv, sizeof(double));
    double* vmass = (double*)calloc((size_t)nv, sizeof(double));
    for (int e = 0; e < m->n_triangles; ++e) {
        const int* tv = m->tri + 3 * e;
        const double area = tri_area(m, e);
        for (int i = 0; i < 3; ++i) vmass[tv[i]] += area / 3.0;
        for (int s = 0; s < 3; ++s) {
            const double* a = m->xy + 2 * tv[s];
            const double* b = m->xy + 2 * tv[(s + 1) % 3];
            const double x = 0.5 * (a[0] + b[0]) - pb->ic_x, y = 0.5 * (a[1] + b[1]) - pb->ic_y;
            const double value = exp(-(x * x + y * y) / pb->ic_w2);
            load[tv[s]] += area / 3.0 * value * 0.5;
            load[tv[(s + 1) % 3]] += area / 3.0 * value * 0.5;
        }
    }
    for (int i = 0; i < op->n; ++i) {
        const int v = op->dof_vertex[i];
        z0[i] = sqrt(vmass[v]) * (load[v] / vmass[v]);
    }
    free(load);
    free(vmass);
}

/* QoI weights: area/3 of every triangle whose centroid lies in the box */
static void qoi_weights(const wmc_oracle_mesh* m, const wmc_oracle_problem* pb, const oper* op, double* w) {
    double* vw = (double*)calloc((size_t)m->n_vertices, sizeof(double));
    for (int e = 0; e < m->n_triangles; ++e) {
        double cx, cy;
        tri_centroid(m, e, &cx, &cy);
        if (cx < pb->box[0] || cx > pb->box[1] || cy < pb->box[2] || cy > pb->box[3]) continue;
        const double area = tri_area(m, e);
        for (int i = 0; i < 3; ++i) vw[m->tri[3 * e + i]] += area / 3.0;
    }
    double total = 0.0;
    for (int v = 0; v < m->n_vertices; ++v) total += vw[v];
    for (int i = 0; i < op->n; ++i) w[i] = pb->qoi_mean ? vw[op->dof_vertex[i]] / total : vw[op->dof_vertex[i]];
    free(vw);
}

int wmc_oracle_level_data(const wmc_oracle_mesh* mesh, const wmc_oracle_problem* pb, double* z0, double* mass,
                          double* qoi_w) {
    double* ones = (double*)malloc(sizeof(double) * (size_t)(pb->cells_x * pb->cells_y));
    for (int k = 0; k < pb->cells_x * pb->cells_y; ++k) ones[k] = 1.0;
    oper op;
    if (build_operator(mesh, pb, ones, &op) != 0) {
        free(ones);
        return -1;
    }
    if (z0) project_z0(mesh, pb, &op, z0);
    if (mass) memcpy(mass, op.mass, sizeof(double) * (size_t)op.n);
    if (qoi_w) qoi_weights(mesh, pb, &op, qoi_w);
    const int n = op.n;
    oper_free(&op);
    free(ones);
    return n;
}

/* ---- power iteration: src/fem.cpp:132-175 (max_eigenvalue), :177-189
 *      (coarse_max_eigenvalue); stable_dt: src/experiments.cpp:30-43 ---- */

/* apply = A (coarse == 0) or the coarse part: x masked on P, A (I-P), rows in P zeroed */
static void eig_apply(const oper* op, int coarse, const double* x, double* y, double* scratch) {
    if (!coarse) {
        csr_mul(&op->a, x, y);
        return;
    }
    for (int i = 0; i < op->n; ++i) scratch[i] = op->sel[i] ? 0.0 : x[i];
    csr_mul(&op->a_coarse, scratch, y);
    for (int i = 0; i < op->n; ++i)
        if (op->sel[i]) y[i] = 0.0;
}

static int power_iteration(const oper* op, int coarse, double tol, int max_iter, const double* warm, double* lambda,
                           double* vec_out, int* iters) {
    const int n = op->n;
    double* v = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* av = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* sc = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    if (warm) {
        memcpy(v, warm, sizeof(double) * (size_t)n);
    } else {
        for (int i = 0; i < n; ++i) v[i] = (double)(wmc_oracle_mix64((uint64_t)i + 1) >> 11) * 0x1.0p-53 - 0.5;
    }
    double norm = 0.0;
    for (int i = 0; i < n; ++i) norm += v[i] * v[i];
    norm = sqrt(norm);
    if (norm == 0.0) {
        v[0] = 1.0;
        norm = 1.0;
    }
    for (int i = 0; i < n; ++i) v[i] /= norm;
    double lambda_prev = 0.0;
    int settled = 0, status = 3;
    for (int it = 1; it <= max_iter; ++it) {
        eig_apply(op, coarse, v, av, sc);
        double rayleigh = 0.0, av2 = 0.0;
        for (int i = 0; i < n; ++i) rayleigh += v[i] * av[i];
        for (int i = 0; i < n; ++i) av2 += av[i] * av[i];
        const double av_norm = sqrt(av2);
        if (iters) *iters = it;
        if (av_norm == 0.0) {
            *lambda = 0.0;
            status = 0;
            break;
        }
        for (int i = 0; i < n; ++i) v[i] = av[i] / av_norm;
        if (fabs(rayleigh - lambda_prev) <= tol * fabs(rayleigh)) {
            if (++settled >= 3) {
                *lambda = rayleigh;
                status = 0;
                break;
            }
        } else {
            settled = 0;
        }
        lambda_prev = rayleigh;
    }
    if (vec_out) memcpy(vec_out, v, sizeof(double) * (size_t)n);
    free(v);
    free(av);
    free(sc);
    return status;
}

static int n_selected(const oper* op) {
    int c = 0;
    for (int i = 0; i < op->n; ++i) c += op->sel[i] != 0;
    return c;
}

static int stable_dt_op(const oper* op, const wmc_oracle_problem* pb, const double* warm_full,
                        const double* warm_coarse, double* dt, int* iters) {
    const double margin = 1.05, tol = 1e-4;
    double lf = 0.0, lc = 0.0;
    int it_f = 0, it_c = 0;
    if (power_iteration(op, 0, tol, 20000, warm_full, &lf, NULL, &it_f) != 0) return 3;
    if (pb->kind == 1 && n_selected(op) > 0) {
        if (power_iteration(op, 1, tol, 20000, warm_coarse, &lc, NULL, &it_c) != 0) return 3;
        int p_fine = pb->substeps;
        for (int k = 1; k < pb->tiers; ++k) p_fine *= pb->substeps;
        const double dt_coarse = 2.0 / sqrt(margin * lc);
        const double dt_fine = p_fine * 2.0 / sqrt(margin * lf);
        *dt = pb->cfl_safety * (dt_coarse < dt_fine ? dt_coarse : dt_fine);
    } else {
        *dt = pb->cfl_safety * 2.0 / sqrt(margin * lf);
    }
    if (iters) {
        iters[0] = it_f;
        iters[1] = it_c;
    }
    return 0;
}

int wmc_oracle_warm_starts(const wmc_oracle_mesh* mesh, const wmc_oracle_problem* pb, double* warm_full,
                           double* warm_coarse) {
    double* ones = (double*)malloc(sizeof(double) * (size_t)(pb->cells_x * pb->cells_y));
    for (int k = 0; k < pb->cells_x * pb->cells_y; ++k) ones[k] = 1.0;
    oper op;
    if (build_operator(mesh, pb, ones, &op) != 0) {
        free(ones);
        return 3;
    }
    double lam;
    int status = power_iteration(&op, 0, 1e-4, 20000, NULL, &lam, warm_full, NULL);
    if (status == 0 && warm_coarse) {
        if (n_selected(&op) > 0)
            status = power_iteration(&op, 1, 1e-4, 20000, NULL, &lam, warm_coarse, NULL);
        else
            memset(warm_coarse, 0, sizeof(double) * (size_t)op.n);
    }
    oper_free(&op);
    free(ones);
    return status;
}

int wmc_oracle_stable_dt(const wmc_oracle_mesh* mesh, const wmc_oracle_problem* pb, const double* cells, double* dt,
                         int* iters) {
    oper op;
    if (build_operator(mesh, pb, cells, &op) != 0) return 3;
    double *wf = NULL, *wc = NULL;
    if (!pb->warm_full) {
        wf = (double*)malloc(sizeof(double) * (size_t)(op.n ? op.n : 1));
        wc = (double*)malloc(sizeof(double) * (size_t)(op.n ? op.n : 1));
        if (wmc_oracle_warm_starts(mesh, pb, wf, wc) != 0) {
            free(wf);
            free(wc);
            oper_free(&op);
            return 3;
        }
    }
    const int status = stable_dt_op(&op, pb, pb->warm_full ? pb->warm_full : wf,
                                    pb->warm_full ? pb->warm_coarse : wc, dt, iters);
    free(wf);
    free(wc);
    oper_free(&op);
    return status;
}

/* ---- time integration: src/integrators.cpp:12-18 (check_finite), :68-87
 *      (leapfrog_init), :89-115 (leapfrog_step), :117-157 (lts_step),
 *      :176-210 (run_wave) ---- */

static int finite_ok(const double* z, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(z[i]) || fabs(z[i]) > 1e100) return 0;
    return 1;
}

/* integrator state shared by the step functions */
typedef struct {
    const oper* op;
    int n, kind, p, tiers;
    double dt, delta, omega;
    double *beta_int, *beta_half;
    csr* a_tier;      /* nested tiers: A P_k, k = 1..tiers (column masks vt >= k) */
    double* buf;      /* scratch */
    long cnt[3];
} integ;

static void integ_init(integ* g, const oper* op, const wmc_oracle_problem* pb, double dt_req) {
    memset(g, 0, sizeof(*g));
    g->op = op;
    g->n = op->n;
    g->kind = pb->kind;
    const long n_steps = (long)ceil(pb->final_time / dt_req - 1e-12);
    g->dt = pb->final_time / (double)n_steps;
    g->p = pb->kind == 1 ? pb->substeps : 1;
    g->tiers = pb->kind == 1 && pb->tiers > 1 ? pb->tiers : 1;
    g->delta = 1.0;
    g->omega = 2.0;
    g->beta_int = (double*)malloc(sizeof(double) * (size_t)(g->p + 1));
    g->beta_half = (double*)malloc(sizeof(double) * (size_t)(g->p + 1));
    if (pb->kind == 1) wmc_oracle_chebyshev(g->p, pb->nu, &g->delta, &g->omega, g->beta_int, g->beta_half);
    if (g->tiers > 1) {
        g->a_tier = (csr*)malloc(sizeof(csr) * (size_t)g->tiers);
        unsigned char* keep = (unsigned char*)malloc((size_t)(g->n ? g->n : 1));
        for (int k = 1; k <= g->tiers; ++k) {
            for (int i = 0; i < g->n; ++i) keep[i] = op->vt[i] >= k;
            g->a_tier[k - 1] = csr_mask(&op->a, keep, 1);
        }
        free(keep);
        /* per tier: rho, rt, E_prev, E_cur, E_next, product */
        g->buf = (double*)malloc(sizeof(double) * (size_t)(g->n ? g->n : 1) * 6 * (size_t)g->tiers);
    }
}

static void integ_free(integ* g) {
    free(g->beta_int);
    free(g->beta_half);
    if (g->a_tier) {
        for (int k = 0; k < g->tiers; ++k) csr_free(&g->a_tier[k]);
        free(g->a_tier);
    }
    free(g->buf);
}

/* Nested LTS (BASELINE config 2; no reference counterpart, parity unpinned
 * by the reference -- pinned by reduction, see tests): tier k advances the
 * local problem e'' = -(r + A P_k e), e(0) = e'(0) = 0, over its interval
 * dt_k = dt / p^(k-1) with the reference's stabilised recursion
 * (src/integrators.cpp:117-157) at step dt_k / p, where the right-hand side
 * of each stage, rho_m = r + A P_k E_m, is replaced by the effective one of
 * tier k+1 over the stage: rt = -2 E^(k+1)_p(rho_m) / dt_(k+1)^2.  The
 * innermost tier uses rho directly.  Returns E^k_p in out. */
static void tier_solve(integ* g, int k, const double* r, double* out) {
    const int n = g->n, p = g->p;
    double* rho = g->buf + (size_t)n * 6 * (size_t)(k - 1);
    double* rt = rho + n;
    double* ep = rt + n;
    double* ec = ep + n;
    double* en = ec + n;
    double* prod = en + n;
    double dt_k = g->dt;
    for (int j = 1; j < k; ++j) dt_k /= p;
    const double tau2 = (dt_k / p) * (dt_k / p);
    const double c0 = 0.5 * tau2 * 2.0 * p * p / (g->omega * g->delta);
    const double dt_child = dt_k / p;
    const double back = -2.0 / (dt_child * dt_child);
    for (int i = 0; i < n; ++i) ep[i] = ec[i] = 0.0;
    for (int m = 0; m < p; ++m) {
        if (m > 0) {
            csr_mul(&g->a_tier[k - 1], ec, prod);
            g->cnt[1]++;
            for (int i = 0; i < n; ++i) rho[i] = r[i] + prod[i];
        } else {
            for (int i = 0; i < n; ++i) rho[i] = r[i];
        }
        if (k < g->tiers) {
            tier_solve(g, k + 1, rho, rt);
            for (int i = 0; i < n; ++i) rt[i] = back * rt[i];
        } else {
            for (int i = 0; i < n; ++i) rt[i] = rho[i];
        }
        if (m == 0) {
            for (int i = 0; i < n; ++i) en[i] = -c0 * rt[i];
        } else {
            const double beta = g->beta_int[m - 1];
            const double cm = tau2 * 2.0 * p * p / g->omega * g->beta_half[m - 1];
            for (int i = 0; i < n; ++i) en[i] = (1.0 + beta) * ec[i] - beta * ep[i] - cm * rt[i];
        }
        for (int i = 0; i < n; ++i) {
            ep[i] = ec[i];
            ec[i] = en[i];
        }
    }
    for (int i = 0; i < n; ++i) out[i] = ec[i];
}

/* one global step (z_prev, z_curr) -> (z_curr, z_next), scratch of 5 n */
static void integ_step(integ* g, double* zp, double* zc, double* s) {
    const int n = g->n, p = g->p;
    const oper* op = g->op;
    double *aq = s, *w = s + n, *az = s + 2 * n, *qp = s + 3 * n, *qc = s + 4 * n;
    if (g->kind == 0) {
        csr_mul(&op->a, zc, aq);
        g->cnt[0]++;
        const double dt2 = g->dt * g->dt;
        for (int i = 0; i < n; ++i) {
            const double next = 2.0 * zc[i] - zp[i] - dt2 * aq[i];
            zp[i] = zc[i];
            zc[i] = next;
        }
    } else if (g->tiers > 1) {
        csr_mul(&op->a, zc, aq);
        g->cnt[0]++;
        tier_solve(g, 1, aq, qc);
        for (int i = 0; i < n; ++i) {
            const double next = 2.0 * zc[i] - zp[i] + 2.0 * qc[i];
            zp[i] = zc[i];
            zc[i] = next;
        }
    } else {
        const double tau2 = (g->dt / p) * (g->dt / p);
        csr_mul(&op->a_coarse, zc, w);
        g->cnt[2]++;
        csr_mul(&op->a_fine, zc, az);
        g->cnt[1]++;
        const double c0 = 0.5 * tau2 * 2.0 * p * p / (g->omega * g->delta);
        for (int i = 0; i < n; ++i) {
            qp[i] = 0.0;
            qc[i] = -c0 * (w[i] + az[i]);
        }
        for (int m = 1; m <= p - 1; ++m) {
            csr_mul(&op->a_fine, qc, aq);
            g->cnt[1]++;
            const double beta = g->beta_int[m - 1];
            const double cm = tau2 * 2.0 * p * p / g->omega * g->beta_half[m - 1];
            for (int i = 0; i < n; ++i) {
                const double next = (1.0 + beta) * qc[i] - beta * qp[i] - cm * (w[i] + az[i] + aq[i]);
                qp[i] = qc[i];
                qc[i] = next;
            }
        }
        for (int i = 0; i < n; ++i) {
            const double next = 2.0 * zc[i] - zp[i] + 2.0 * qc[i];
            zp[i] = zc[i];
            zc[i] = next;
        }
    }
}

int wmc_oracle_solve(const wmc_oracle_mesh* mesh, const wmc_oracle_problem* pb, const double* cells, double* q,
                     long* fail_step, long* counters) {
    oper op;
    if (build_operator(mesh, pb, cells, &op) != 0) return 3;
    const int n = op.n;
    const size_t bytes = sizeof(double) * (size_t)(n ? n : 1);
    double* z0 = (double*)malloc(bytes);
    double* zp = (double*)malloc(bytes);
    double* zc = (double*)malloc(bytes);
    double* scratch = (double*)malloc(bytes * 5);
    double* qw = (double*)malloc(bytes);
    int status = 0;
    project_z0(mesh, pb, &op, z0);
    qoi_weights(mesh, pb, &op, qw);
    /* requested step: fixed, or the sample's stable_dt (run_wave snaps it) */
    double dt_req = pb->dt;
    if (pb->cfl_safety > 0.0) {
        double *wf = NULL, *wc = NULL;
        if (!pb->warm_full) {
            wf = (double*)malloc(bytes);
            wc = (double*)malloc(bytes);
            wmc_oracle_warm_starts(mesh, pb, wf, wc);
        }
        status = stable_dt_op(&op, pb, pb->warm_full ? pb->warm_full : wf, pb->warm_full ? pb->warm_coarse : wc,
                              &dt_req, NULL);
        free(wf);
        free(wc);
        if (status != 0) {
            if (fail_step) *fail_step = 0;
            free(z0);
            free(zp);
            free(zc);
            free(scratch);
            free(qw);
            oper_free(&op);
            return status;
        }
    }
    integ g;
    integ_init(&g, &op, pb, dt_req);
    const long n_steps = (long)ceil(pb->final_time / dt_req - 1e-12);
    const double dt = g.dt;

    /* leapfrog_init: z1 = z0 + dt M^{1/2} v0 + dt^2/2 (F0 - A z0), v0 = F = 0 */
    csr_mul(&op.a, z0, scratch);
    g.cnt[0]++;
    for (int i = 0; i < n; ++i) {
        zp[i] = z0[i];
        zc[i] = z0[i] + dt * 0.0 + 0.5 * dt * dt * (0.0 - scratch[i]);
    }
    long step = 1;
    if (!finite_ok(zc, n)) status = 3;
    for (long s = 1; s < n_steps && status == 0; ++s) {
        integ_step(&g, zp, zc, scratch);
        ++step;
        if (!finite_ok(zc, n)) status = 3;
    }
    if (status == 0) {
        /* Q = sum_i w_i u_i, u = z / sqrt(M) (fem.cpp:271-275) */
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += qw[i] * (zc[i] / sqrt(op.mass[i]));
        *q = acc;
    } else if (fail_step) {
        *fail_step = step;
    }
    if (counters) {
        counters[0] = g.cnt[0];
        counters[1] = g.cnt[1];
        counters[2] = g.cnt[2];
    }
    integ_free(&g);
    free(z0);
    free(zp);
    free(zc);
    free(scratch);
    free(qw);
    oper_free(&op);
    return status;
}

int wmc_oracle_steps(const wmc_oracle_mesh* mesh, const wmc_oracle_problem* pb, const double* cells, double* z_prev,
                     double* z_curr, long n_steps) {
    oper op;
    if (build_operator(mesh, pb, cells, &op) != 0) return 3;
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(op.n ? op.n : 1) * 5);
    integ g;
    integ_init(&g, &op, pb, pb->dt);
    int status = 0;
    for (long s = 0; s < n_steps && status == 0; ++s) {
        integ_step(&g, z_prev, z_curr, scratch);
        if (!finite_ok(z_curr, op.n)) status = 3;
    }
    integ_free(&g);
    free(scratch);
    oper_free(&op);
    return status;
}

/* ---- MLMC: src/mlmc.cpp:21-37 (sample_delta_q), :44-73 (accumulators) ---- */

int wmc_oracle_eval_pairs(const wmc_oracle_mesh* fine, const wmc_oracle_problem* pf, const wmc_oracle_mesh* coarse,
                          const wmc_oracle_problem* pc, uint64_t seed, uint32_t level, uint64_t first, long count,
                          double* dq, double* q_fine, long* fail_index, long* fail_step) {
    const int ncell = pf->cells_x * pf->cells_y;
    double* cells = (double*)malloc(sizeof(double) * (size_t)ncell);
    int status = 0;
    /* per-level warm starts, once per call (the reference's level contexts) */
    wmc_oracle_problem fpb = *pf, cpb;
    double *wbuf[4] = {NULL, NULL, NULL, NULL};
    if (pf->cfl_safety > 0.0 && !pf->warm_full) {
        int nf = 0;
        for (int v = 0; v < fine->n_vertices; ++v) nf += !fine->boundary[v];
        wbuf[0] = (double*)malloc(sizeof(double) * (size_t)(nf ? nf : 1));
        wbuf[1] = (double*)malloc(sizeof(double) * (size_t)(nf ? nf : 1));
        wmc_oracle_warm_starts(fine, pf, wbuf[0], wbuf[1]);
        fpb.warm_full = wbuf[0];
        fpb.warm_coarse = wbuf[1];
    }
    if (coarse) {
        cpb = *pc;
        if (pc->cfl_safety > 0.0 && !pc->warm_full) {
            int nc = 0;
            for (int v = 0; v < coarse->n_vertices; ++v) nc += !coarse->boundary[v];
            wbuf[2] = (double*)malloc(sizeof(double) * (size_t)(nc ? nc : 1));
            wbuf[3] = (double*)malloc(sizeof(double) * (size_t)(nc ? nc : 1));
            wmc_oracle_warm_starts(coarse, pc, wbuf[2], wbuf[3]);
            cpb.warm_full = wbuf[2];
            cpb.warm_coarse = wbuf[3];
        }
        pc = &cpb;
    }
    pf = &fpb;
    for (long i = 0; i < count && status == 0; ++i) {
        if (pf->kl_table)
            wmc_oracle_draw_kl(seed, level, first + (uint64_t)i, pf->kl_table, ncell, pf->kl_modes, cells);
        else
            wmc_oracle_draw_cells(seed, level, first + (uint64_t)i, ncell, pf->coef_lo, pf->coef_hi, cells);
        double qf = 0.0, qc = 0.0;
        long step = 0;
        status = wmc_oracle_solve(fine, pf, cells, &qf, &step, NULL);
        if (status == 0 && coarse) status = wmc_oracle_solve(coarse, pc, cells, &qc, &step, NULL);
        if (status != 0) {
            if (fail_index) *fail_index = (long)first + i;
            if (fail_step) *fail_step = step;
            break;
        }
        q_fine[i] = qf;
        dq[i] = coarse ? qf - qc : qf;
    }
    for (int k = 0; k < 4; ++k) free(wbuf[k]);
    free(cells);
    return status;
}

void wmc_oracle_moments(const double* dq, const double* q, long n, double* out) {
    /* QoIVector norm on the 2-point grid {0,2} is |value| (tests/test_mlmc.cpp:16-20) */
    double s_dq = 0.0, s_dq2 = 0.0, s_q = 0.0, s_q2 = 0.0;
    for (long i = 0; i < n; ++i) {
        const double a = fabs(dq[i]), b = fabs(q[i]);
        s_dq2 += a * a;
        s_q2 += b * b;
        s_dq += dq[i];
        s_q += q[i];
    }
    const double nn = (double)n;
    double var = 0.0, mcvar = 0.0;
    if (n >= 2) {
        const double sn = fabs(s_dq), qn = fabs(s_q);
        var = (s_dq2 - sn * sn / nn) / (nn - 1.0);
        mcvar = (s_q2 - qn * qn / nn) / nn;
        if (var < 0.0) var = 0.0;
        if (mcvar < 0.0) mcvar = 0.0;
    }
    out[0] = nn;
    out[1] = s_dq;
    out[2] = s_dq2;
    out[3] = s_q;
    out[4] = s_q2;
    out[5] = var;
    out[6] = mcvar;
}
