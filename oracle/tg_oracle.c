/* TEST INFRASTRUCTURE ONLY — see tg_oracle.h.
 *
 * Plain-C restatement of the reference P1 assembly path.  Floating-point
 * expressions are written in the reference's evaluation order and compiled
 * with -ffp-contract=off, so every value is bit-identical to libtg (which is
 * built without -march and therefore contains no FMA).
 * Citations are /root/reference/proj/<file>:<line>.
 */
#include "tg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];

const char* tgo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* reference.cpp:18-34 */
int tgo_element_dim(int kind) { return kind == TGO_TET4 ? 3 : 2; }
int tgo_element_nodes(int kind) { return kind == TGO_TRI3 ? 3 : 4; }
/* reference.cpp:241-247 */
int tgo_default_degree(int kind, int mass) {
    if (kind == TGO_QUAD4) return 3;
    return mass ? 2 : 1;
}
static int is_affine(int kind) { return kind != TGO_QUAD4; } /* batch.cpp:16 */

/* ReferenceElement::shape_values / shape_gradients (reference.cpp:45-71) */
static void shape_values(int kind, const double* p, double* v) {
    if (kind == TGO_TRI3) {
        v[0] = 1.0 - p[0] - p[1];
        v[1] = p[0];
        v[2] = p[1];
    } else if (kind == TGO_QUAD4) {
        const double x = p[0], y = p[1];
        v[0] = (1 - x) * (1 - y);
        v[1] = x * (1 - y);
        v[2] = x * y;
        v[3] = (1 - x) * y;
    } else {
        v[0] = 1.0 - p[0] - p[1] - p[2];
        v[1] = p[0];
        v[2] = p[1];
        v[3] = p[2];
    }
}

static void shape_gradients(int kind, const double* p, double* g) {
    if (kind == TGO_TRI3) {
        const double t[6] = {-1, -1, 1, 0, 0, 1};
        memcpy(g, t, sizeof t);
    } else if (kind == TGO_QUAD4) {
        const double x = p[0], y = p[1];
        const double t[8] = {-(1 - y), -(1 - x), (1 - y), -x, y, x, -y, (1 - x)};
        memcpy(g, t, sizeof t);
    } else {
        const double t[12] = {-1, -1, -1, 1, 0, 0, 0, 1, 0, 0, 0, 1};
        memcpy(g, t, sizeof t);
    }
}

/* quadrature rules: tri_rule (reference.cpp:99-132), quad_rule (:134-166),
 * tet_rule (:168-210) */
static int rule(int kind, int degree, int* Q, double* pts, double* w) {
    if (degree < 1 || degree > 4) return fail(2, "quadrature degree unsupported; supported degrees: 1,2,3,4");
    if (kind == TGO_TRI3) {
        if (degree == 1) {
            *Q = 1;
            pts[0] = 1.0 / 3.0; pts[1] = 1.0 / 3.0;
            w[0] = 0.5;
        } else if (degree == 2) {
            const double p[6] = {1.0 / 6, 1.0 / 6, 2.0 / 3, 1.0 / 6, 1.0 / 6, 2.0 / 3};
            *Q = 3;
            memcpy(pts, p, sizeof p);
            w[0] = w[1] = w[2] = 1.0 / 6;
        } else if (degree == 3) {
            const double p[8] = {1.0 / 3, 1.0 / 3, 0.2, 0.2, 0.6, 0.2, 0.2, 0.6};
            const double ww[4] = {-27.0 / 96, 25.0 / 96, 25.0 / 96, 25.0 / 96};
            *Q = 4;
            memcpy(pts, p, sizeof p);
            memcpy(w, ww, sizeof ww);
        } else {
            const double a1 = 0.445948490915965, w1 = 0.223381589678011;
            const double a2 = 0.091576213509771, w2 = 0.109951743655322;
            const double p[12] = {a1, a1, 1 - 2 * a1, a1, a1, 1 - 2 * a1,
                                  a2, a2, 1 - 2 * a2, a2, a2, 1 - 2 * a2};
            *Q = 6;
            memcpy(pts, p, sizeof p);
            for (int i = 0; i < 3; ++i) w[i] = w1 / 2;
            for (int i = 3; i < 6; ++i) w[i] = w2 / 2;
        }
    } else if (kind == TGO_QUAD4) {
        double g[3], gw[3];
        int n;
        if (degree <= 1) {
            n = 1; g[0] = 0.5; gw[0] = 1.0;
        } else if (degree <= 3) {
            const double s = 0.5 / sqrt(3.0);
            n = 2; g[0] = 0.5 - s; g[1] = 0.5 + s; gw[0] = 0.5; gw[1] = 0.5;
        } else {
            const double s = 0.5 * sqrt(0.6);
            n = 3; g[0] = 0.5 - s; g[1] = 0.5; g[2] = 0.5 + s;
            gw[0] = 5.0 / 18; gw[1] = 8.0 / 18; gw[2] = 5.0 / 18;
        }
        *Q = n * n;
        int q = 0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i, ++q) {
                pts[2 * q] = g[i];
                pts[2 * q + 1] = g[j];
                w[q] = gw[i] * gw[j];
            }
    } else {
        if (degree == 1) {
            *Q = 1;
            pts[0] = pts[1] = pts[2] = 0.25;
            w[0] = 1.0 / 6.0;
        } else if (degree == 2) {
            const double a = 0.585410196624969, b = 0.138196601125011;
            const double p[12] = {b, b, b, a, b, b, b, a, b, b, b, a};
            *Q = 4;
            memcpy(pts, p, sizeof p);
            for (int i = 0; i < 4; ++i) w[i] = 1.0 / 24.0;
        } else if (degree == 3) {
            const double s = 1.0 / 6.0;
            const double p[15] = {0.25, 0.25, 0.25, s, s, s, 0.5, s, s, s, 0.5, s, s, s, 0.5};
            *Q = 5;
            memcpy(pts, p, sizeof p);
            w[0] = -4.0 / 5.0 / 6.0;
            for (int i = 1; i < 5; ++i) w[i] = 9.0 / 20.0 / 6.0;
        } else {
            const double a = 11.0 / 14.0, b = 1.0 / 14.0;
            const double c = 0.399403576166799, dd = 0.100596423833201;
            const double w1 = -74.0 / 5625.0, w2 = 343.0 / 45000.0, w3 = 56.0 / 2250.0;
            const double p[33] = {0.25, 0.25, 0.25, b, b, b, a, b, b, b, a, b, b, b, a,
                                  c, dd, dd, dd, c, dd, dd, dd, c, dd, c, c, c, dd, c, c, c, dd};
            const double ww[11] = {w1, w2, w2, w2, w2, w3, w3, w3, w3, w3, w3};
            *Q = 11;
            memcpy(pts, p, sizeof p);
            memcpy(w, ww, sizeof ww);
        }
    }
    return 0;
}

#define MAXQ 11
typedef struct {
    int kind, k, d, Q;
    double pts[MAXQ * 3], w[MAXQ], B[MAXQ * 4], G[MAXQ * 4 * 3];
} tables_t;

/* reference_tables (reference.cpp:223-239) */
static int make_tables(int kind, int degree, tables_t* t) {
    t->kind = kind;
    t->k = tgo_element_nodes(kind);
    t->d = tgo_element_dim(kind);
    int rc = rule(kind, degree, &t->Q, t->pts, t->w);
    if (rc) return rc;
    for (int q = 0; q < t->Q; ++q) {
        double v[4], g[12];
        shape_values(kind, &t->pts[q * t->d], v);
        shape_gradients(kind, &t->pts[q * t->d], g);
        for (int a = 0; a < t->k; ++a) {
            t->B[q * t->k + a] = v[a];
            for (int c = 0; c < t->d; ++c) t->G[(q * t->k + a) * t->d + c] = g[a * t->d + c];
        }
    }
    return 0;
}

int tgo_tables(int kind, int degree, int* Q, double* points, double* weights, double* B,
               double* G) {
    tables_t t;
    int rc = make_tables(kind, degree, &t);
    if (rc) return rc;
    *Q = t.Q;
    if (points) memcpy(points, t.pts, sizeof(double) * t.Q * t.d);
    if (weights) memcpy(weights, t.w, sizeof(double) * t.Q);
    if (B) memcpy(B, t.B, sizeof(double) * t.Q * t.k);
    if (G) memcpy(G, t.G, sizeof(double) * t.Q * t.k * t.d);
    return 0;
}

/* ------------------------------------------------------------------ mesh */

void tgo_grid_sizes(int kind, const int64_t* div, int64_t* n_nodes, int64_t* n_elems) {
    if (kind == TGO_TET4) {
        *n_nodes = (div[0] + 1) * (div[1] + 1) * (div[2] + 1);
        *n_elems = 6 * div[0] * div[1] * div[2];
    } else {
        *n_nodes = (div[0] + 1) * (div[1] + 1);
        *n_elems = (kind == TGO_TRI3 ? 2 : 1) * div[0] * div[1];
    }
}

/* centroid_det (mesh.cpp:31-52) */
static double centroid_det(int kind, const double* nodes, const int64_t* conn) {
    const int k = tgo_element_nodes(kind), d = tgo_element_dim(kind);
    double centroid[3] = {0, 0, 0};
    static const double ref_nodes[3][4][3] = {
        {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 0}},
        {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}},
        {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
    for (int a = 0; a < k; ++a)
        for (int c = 0; c < d; ++c) centroid[c] += ref_nodes[kind][a][c] / k;
    double g[12];
    shape_gradients(kind, centroid, g);
    double J[3][3] = {{0}};
    for (int a = 0; a < k; ++a) {
        const double* x = &nodes[conn[a] * d];
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) J[i][j] += x[i] * g[a * d + j];
    }
    if (d == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

/* generate_grid (mesh.cpp:96-169) */
int tgo_generate_grid(int kind, const double* ext, const int64_t* div, double* nodes,
                      int64_t* elems) {
    const int d = tgo_element_dim(kind);
    for (int c = 0; c < d; ++c)
        if (div[c] < 1) return fail(2, "generate_grid: divisions must be >= 1");
    if (d == 2) {
        const int64_t nx = div[0], ny = div[1];
        const double hx = ext[0] / nx, hy = ext[1] / ny;
        int64_t p = 0;
        for (int64_t j = 0; j <= ny; ++j)
            for (int64_t i = 0; i <= nx; ++i) {
                nodes[p++] = i * hx;
                nodes[p++] = j * hy;
            }
        int64_t q = 0;
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t n00 = i + j * (nx + 1), n10 = (i + 1) + j * (nx + 1);
                const int64_t n11 = (i + 1) + (j + 1) * (nx + 1), n01 = i + (j + 1) * (nx + 1);
                if (kind == TGO_QUAD4) {
                    elems[q++] = n00; elems[q++] = n10; elems[q++] = n11; elems[q++] = n01;
                } else {
                    elems[q++] = n00; elems[q++] = n10; elems[q++] = n11;
                    elems[q++] = n00; elems[q++] = n11; elems[q++] = n01;
                }
            }
    } else {
        const int64_t nx = div[0], ny = div[1], nz = div[2];
        const double hx = ext[0] / nx, hy = ext[1] / ny, hz = ext[2] / nz;
        int64_t p = 0;
        for (int64_t kz = 0; kz <= nz; ++kz)
            for (int64_t j = 0; j <= ny; ++j)
                for (int64_t i = 0; i <= nx; ++i) {
                    nodes[p++] = i * hx;
                    nodes[p++] = j * hy;
                    nodes[p++] = kz * hz;
                }
        static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                        {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        int64_t e = 0;
        for (int64_t kz = 0; kz < nz; ++kz)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t i = 0; i < nx; ++i)
                    for (int s6 = 0; s6 < 6; ++s6, ++e) {
                        int64_t c[3] = {0, 0, 0};
                        int64_t* tet = &elems[e * 4];
                        tet[0] = i + (nx + 1) * (j + (ny + 1) * kz);
                        for (int s = 0; s < 3; ++s) {
                            c[perms[s6][s]] = 1;
                            tet[s + 1] = (i + c[0]) + (nx + 1) * ((j + c[1]) + (ny + 1) * (kz + c[2]));
                        }
                        if (centroid_det(kind, nodes, tet) < 0.0) {
                            const int64_t tmp = tet[2];
                            tet[2] = tet[3];
                            tet[3] = tmp;
                        }
                    }
    }
    return 0;
}

/* Mesh::content_hash (mesh.cpp:79-94), FNV-1a */
static uint64_t fnv(uint64_t h, const void* data, size_t n) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

uint64_t tgo_content_hash(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                          int64_t n_elems) {
    const int d = tgo_element_dim(kind), k = tgo_element_nodes(kind);
    uint64_t h = 14695981039346656037ull;
    const int kind_tag = kind, dim = d;
    h = fnv(h, &kind_tag, sizeof kind_tag);
    h = fnv(h, &dim, sizeof dim);
    h = fnv(h, nodes, (size_t)n_nodes * d * sizeof(double));
    h = fnv(h, elems, (size_t)n_elems * k * sizeof(int64_t));
    return h;
}

/* build_dofmap (dofmap.cpp:9-25) */
void tgo_dofmap(int kind, const int64_t* elems, int64_t n_elems, int comps, int64_t* map) {
    const int kg = tgo_element_nodes(kind), k = kg * comps;
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < kg; ++a)
            for (int c = 0; c < comps; ++c) map[e * k + a * comps + c] = elems[e * kg + a] * comps + c;
}

/* ------------------------------------------------------------------ map */

/* invert_transpose (batch.cpp:18-46) */
static void invert_transpose(const double* J, double det, int d, double* out) {
    if (d == 2) {
        out[0] = J[3] / det;
        out[1] = -J[2] / det;
        out[2] = -J[1] / det;
        out[3] = J[0] / det;
    } else {
        const double c00 = J[4] * J[8] - J[5] * J[7];
        const double c01 = J[5] * J[6] - J[3] * J[8];
        const double c02 = J[3] * J[7] - J[4] * J[6];
        const double c10 = J[2] * J[7] - J[1] * J[8];
        const double c11 = J[0] * J[8] - J[2] * J[6];
        const double c12 = J[1] * J[6] - J[0] * J[7];
        const double c20 = J[1] * J[5] - J[2] * J[4];
        const double c21 = J[2] * J[3] - J[0] * J[5];
        const double c22 = J[0] * J[4] - J[1] * J[3];
        out[0] = c00 / det; out[1] = c01 / det; out[2] = c02 / det;
        out[3] = c10 / det; out[4] = c11 / det; out[5] = c12 / det;
        out[6] = c20 / det; out[7] = c21 / det; out[8] = c22 / det;
    }
}

typedef struct {
    int64_t E;
    int Q, k, d;
    double *jac, *det, *jinv, *qp, *G;
} geom_t;

static void geom_free(geom_t* g) {
    free(g->jac); free(g->det); free(g->jinv); free(g->qp); free(g->G);
}

/* batch_geometry (batch.cpp:56-128) + push_forward (batch.cpp:130-154) */
static int geometry(const tables_t* t, const double* nodes, const int64_t* elems, int64_t E,
                    geom_t* g, int64_t* bad) {
    const int Q = t->Q, k = t->k, d = t->d;
    g->E = E; g->Q = Q; g->k = k; g->d = d;
    g->jac = malloc(sizeof(double) * (size_t)E * Q * d * d + 8);
    g->det = malloc(sizeof(double) * (size_t)E * Q + 8);
    g->jinv = malloc(sizeof(double) * (size_t)E * Q * d * d + 8);
    g->qp = malloc(sizeof(double) * (size_t)E * Q * d + 8);
    g->G = malloc(sizeof(double) * (size_t)E * Q * k * d + 8);
    const int affine = is_affine(t->kind);
    int64_t first_bad = -1;
    for (int64_t e = 0; e < E; ++e) {
        const int64_t* conn = &elems[e * k];
        double X[12];
        for (int a = 0; a < k; ++a)
            for (int c = 0; c < d; ++c) X[a * d + c] = nodes[conn[a] * d + c];
        const int q_eval = affine ? 1 : Q;
        for (int q = 0; q < q_eval; ++q) {
            double* J = &g->jac[((size_t)e * Q + q) * d * d];
            for (int i = 0; i < d * d; ++i) J[i] = 0.0;
            const double* Gh = &t->G[q * k * d];
            for (int a = 0; a < k; ++a)
                for (int i = 0; i < d; ++i)
                    for (int j = 0; j < d; ++j) J[i * d + j] += X[a * d + i] * Gh[a * d + j];
            double det;
            if (d == 2)
                det = J[0] * J[3] - J[1] * J[2];
            else
                det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                      J[2] * (J[3] * J[7] - J[4] * J[6]);
            if (det <= 0.0) {
                if (first_bad < 0) first_bad = e;
                det = 1.0; /* keep going; reported below */
            }
            g->det[(size_t)e * Q + q] = det;
            invert_transpose(J, det, d, &g->jinv[((size_t)e * Q + q) * d * d]);
        }
        if (affine)
            for (int q = 1; q < Q; ++q) {
                memcpy(&g->jac[((size_t)e * Q + q) * d * d], &g->jac[(size_t)e * Q * d * d], sizeof(double) * d * d);
                memcpy(&g->jinv[((size_t)e * Q + q) * d * d], &g->jinv[(size_t)e * Q * d * d], sizeof(double) * d * d);
                g->det[(size_t)e * Q + q] = g->det[(size_t)e * Q];
            }
        for (int q = 0; q < Q; ++q) {
            double* xq = &g->qp[((size_t)e * Q + q) * d];
            for (int c = 0; c < d; ++c) xq[c] = 0.0;
            const double* B = &t->B[q * k];
            for (int a = 0; a < k; ++a)
                for (int c = 0; c < d; ++c) xq[c] += B[a] * X[a * d + c];
        }
        for (int q = 0; q < Q; ++q) {
            const double* JiT = &g->jinv[((size_t)e * Q + q) * d * d];
            const double* Gh = &t->G[q * k * d];
            double* out = &g->G[((size_t)e * Q + q) * k * d];
            for (int a = 0; a < k; ++a)
                for (int i = 0; i < d; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < d; ++j) s += JiT[i * d + j] * Gh[a * d + j];
                    out[a * d + i] = s;
                }
        }
    }
    if (first_bad >= 0) {
        if (bad) *bad = first_bad;
        char msg[128];
        snprintf(msg, sizeof msg, "element %lld has non-positive Jacobian determinant", (long long)first_bad);
        geom_free(g);
        return fail(2, msg);
    }
    return 0;
}

int tgo_geometry(int kind, const double* nodes, const int64_t* elems, int64_t n_elems,
                 int degree, double* jac, double* det, double* jac_invT, double* qpts,
                 double* grads, int64_t* bad) {
    tables_t t;
    int rc = make_tables(kind, degree, &t);
    if (rc) return rc;
    geom_t g;
    rc = geometry(&t, nodes, elems, n_elems, &g, bad);
    if (rc) return rc;
    const size_t EQ = (size_t)n_elems * t.Q;
    if (jac) memcpy(jac, g.jac, EQ * t.d * t.d * 8);
    if (det) memcpy(det, g.det, EQ * 8);
    if (jac_invT) memcpy(jac_invT, g.jinv, EQ * t.d * t.d * 8);
    if (qpts) memcpy(qpts, g.qp, EQ * t.d * 8);
    if (grads) memcpy(grads, g.G, EQ * t.k * t.d * 8);
    geom_free(&g);
    return 0;
}

/* local_stiffness_diffusion (batch.cpp:156-181) */
static void k_diffusion(const tables_t* t, const geom_t* g, const double* coeff, double* K) {
    const int Q = g->Q, k = g->k, d = g->d;
    for (int64_t e = 0; e < g->E; ++e) {
        double* Ke = &K[(size_t)e * k * k];
        for (int i = 0; i < k * k; ++i) Ke[i] = 0.0;
        for (int q = 0; q < Q; ++q) {
            const double scale = t->w[q] * g->det[(size_t)e * Q + q] * coeff[(size_t)e * Q + q];
            const double* G = &g->G[((size_t)e * Q + q) * k * d];
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) {
                    double dot = 0.0;
                    for (int c = 0; c < d; ++c) dot += G[a * d + c] * G[b * d + c];
                    Ke[a * k + b] += scale * dot;
                }
        }
    }
}

/* local_stiffness_elasticity (batch.cpp:183-248) */
static int k_elasticity(const tables_t* t, const geom_t* g, const double* lam_eq,
                        const double* mu_eq, double* K) {
    const int Q = g->Q, kg = g->k, d = g->d, k = kg * d;
    const int ns = d == 2 ? 3 : 6;
    for (size_t i = 0; i < (size_t)g->E * Q; ++i)
        if (mu_eq[i] <= 0.0) return fail(2, "elasticity requires mu > 0");
    double B[6 * 12], DB[6 * 12];
    for (int64_t e = 0; e < g->E; ++e) {
        double* Ke = &K[(size_t)e * k * k];
        for (int i = 0; i < k * k; ++i) Ke[i] = 0.0;
        for (int q = 0; q < Q; ++q) {
            const double* G = &g->G[((size_t)e * Q + q) * kg * d];
            for (int i = 0; i < ns * k; ++i) B[i] = 0.0;
            if (d == 2) {
                for (int a = 0; a < kg; ++a) {
                    const double gx = G[a * 2 + 0], gy = G[a * 2 + 1];
                    B[0 * k + a * 2 + 0] = gx;
                    B[1 * k + a * 2 + 1] = gy;
                    B[2 * k + a * 2 + 0] = gy;
                    B[2 * k + a * 2 + 1] = gx;
                }
            } else {
                for (int a = 0; a < kg; ++a) {
                    const double gx = G[a * 3 + 0], gy = G[a * 3 + 1], gz = G[a * 3 + 2];
                    B[0 * k + a * 3 + 0] = gx;
                    B[1 * k + a * 3 + 1] = gy;
                    B[2 * k + a * 3 + 2] = gz;
                    B[3 * k + a * 3 + 0] = gy;
                    B[3 * k + a * 3 + 1] = gx;
                    B[4 * k + a * 3 + 1] = gz;
                    B[4 * k + a * 3 + 2] = gy;
                    B[5 * k + a * 3 + 0] = gz;
                    B[5 * k + a * 3 + 2] = gx;
                }
            }
            const double lam = lam_eq[(size_t)e * Q + q], mu = mu_eq[(size_t)e * Q + q];
            const int nn = d;
            for (int col = 0; col < k; ++col) {
                double tr = 0.0;
                for (int i = 0; i < nn; ++i) tr += B[i * k + col];
                for (int i = 0; i < nn; ++i) DB[i * k + col] = lam * tr + 2.0 * mu * B[i * k + col];
                for (int i = nn; i < ns; ++i) DB[i * k + col] = mu * B[i * k + col];
            }
            const double scale = t->w[q] * g->det[(size_t)e * Q + q];
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) {
                    double s = 0.0;
                    for (int i = 0; i < ns; ++i) s += B[i * k + a] * DB[i * k + b];
                    Ke[a * k + b] += scale * s;
                }
        }
    }
    return 0;
}

/* local_mass (batch.cpp:250-269) */
static void k_mass(const tables_t* t, const geom_t* g, const double* coeff, double* M) {
    const int Q = g->Q, k = g->k;
    for (int64_t e = 0; e < g->E; ++e) {
        double* Me = &M[(size_t)e * k * k];
        for (int i = 0; i < k * k; ++i) Me[i] = 0.0;
        for (int q = 0; q < Q; ++q) {
            const double scale = t->w[q] * g->det[(size_t)e * Q + q] * coeff[(size_t)e * Q + q];
            const double* B = &t->B[q * k];
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) Me[a * k + b] += scale * B[a] * B[b];
        }
    }
}

/* local_load (batch.cpp:271-289) */
static void k_load(const tables_t* t, const geom_t* g, const double* src, double* F) {
    const int Q = g->Q, k = g->k;
    for (int64_t e = 0; e < g->E; ++e) {
        double* Fe = &F[(size_t)e * k];
        for (int a = 0; a < k; ++a) Fe[a] = 0.0;
        for (int q = 0; q < Q; ++q) {
            const double scale = t->w[q] * g->det[(size_t)e * Q + q] * src[(size_t)e * Q + q];
            const double* B = &t->B[q * k];
            for (int a = 0; a < k; ++a) Fe[a] += scale * B[a];
        }
    }
}

/* local_load_vector (batch.cpp:291-312) */
static void k_load_vector(const tables_t* t, const geom_t* g, const double* src, double* F) {
    const int Q = g->Q, kg = g->k, d = g->d;
    for (int64_t e = 0; e < g->E; ++e) {
        double* Fe = &F[(size_t)e * kg * d];
        for (int a = 0; a < kg * d; ++a) Fe[a] = 0.0;
        for (int q = 0; q < Q; ++q) {
            const double scale = t->w[q] * g->det[(size_t)e * Q + q];
            const double* B = &t->B[q * kg];
            const double* f = &src[((size_t)e * Q + q) * d];
            for (int a = 0; a < kg; ++a)
                for (int c = 0; c < d; ++c) Fe[a * d + c] += scale * B[a] * f[c];
        }
    }
}

static int run_local(const tables_t* t, const geom_t* g, int what, const double* c1,
                     const double* c2, double* out) {
    switch (what) {
        case TGO_DIFFUSION: k_diffusion(t, g, c1, out); return 0;
        case TGO_ELASTICITY: return k_elasticity(t, g, c1, c2, out);
        case TGO_MASS: k_mass(t, g, c1, out); return 0;
        case TGO_LOAD: k_load(t, g, c1, out); return 0;
        case TGO_LOAD_VECTOR: k_load_vector(t, g, c1, out); return 0;
    }
    return fail(2, "unknown local kernel");
}

int tgo_local(int kind, const double* nodes, const int64_t* elems, int64_t n_elems, int degree,
              int what, const double* c1, const double* c2, double* out, int64_t* bad) {
    tables_t t;
    int rc = make_tables(kind, degree, &t);
    if (rc) return rc;
    geom_t g;
    rc = geometry(&t, nodes, elems, n_elems, &g, bad);
    if (rc) return rc;
    rc = run_local(&t, &g, what, c1, c2, out);
    geom_free(&g);
    return rc;
}

/* CoefficientField::evaluate (coefficient.cpp:34-55); nodal via interpolate_nodal
 * (batch.cpp:314-333) */
static int evaluate(const tables_t* t, const int64_t* elems, int64_t E, int64_t n_nodes,
                    const tgo_field* f, double* out) {
    const int Q = t->Q, k = t->k;
    if (f->type == 0) {
        for (size_t i = 0; i < (size_t)E * Q; ++i) out[i] = f->value;
    } else if (f->type == 1) {
        if (f->n != E) return fail(2, "per-element coefficient: wrong number of values");
        for (int64_t e = 0; e < E; ++e)
            for (int q = 0; q < Q; ++q) out[(size_t)e * Q + q] = f->data[e];
    } else if (f->type == 2) {
        if (f->n != n_nodes) return fail(2, "nodal field: wrong number of values");
        for (int64_t e = 0; e < E; ++e) {
            const int64_t* conn = &elems[e * k];
            for (int q = 0; q < Q; ++q) {
                const double* B = &t->B[q * k];
                double s = 0.0;
                for (int a = 0; a < k; ++a) s += B[a] * f->data[conn[a]];
                out[(size_t)e * Q + q] = s;
            }
        }
    } else {
        return fail(2, "unknown field type");
    }
    return 0;
}

int tgo_evaluate(int kind, const double* nodes, const int64_t* elems, int64_t n_elems,
                 int64_t n_nodes, int degree, const tgo_field* f, double* out) {
    (void)nodes;
    tables_t t;
    int rc = make_tables(kind, degree, &t);
    if (rc) return rc;
    return evaluate(&t, elems, n_elems, n_nodes, f, out);
}

/* ------------------------------------------------------------------ routing */

struct tgo_routing {
    int64_t N, E, nnz;
    int k;
    int64_t *offsets, *cols;
    uint32_t *vec_off, *vec_slots, *mat_off, *mat_slots;
};

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* CsrPattern::find (sparse.cpp:10-16) */
static int64_t find(const tgo_routing* r, int64_t i, int64_t j) {
    int64_t lo = r->offsets[i], hi = r->offsets[i + 1];
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (r->cols[mid] < j) lo = mid + 1; else hi = mid;
    }
    if (lo == r->offsets[i + 1] || r->cols[lo] != j) return -1;
    return lo;
}

/* build_routing (routing.cpp:12-85).  The pattern (sorted unique (g_a,g_b)
 * pairs, routing.cpp:17-36) is formed per row — the same set, hence the same
 * CSR — then the segment maps exactly as routing.cpp:47-83. */
tgo_routing* tgo_routing_build(int64_t N, int64_t E, int k, const int64_t* map) {
    if (E * (int64_t)k * k > (int64_t)UINT32_MAX) {
        fail(2, "build_routing: mesh exceeds 2^32-1 local matrix slots");
        return NULL;
    }
    tgo_routing* r = calloc(1, sizeof *r);
    r->N = N; r->E = E; r->k = k;
    /* candidate columns per row */
    int64_t* cnt = calloc((size_t)N + 1, sizeof(int64_t));
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a) cnt[map[e * k + a] + 1] += k;
    for (int64_t i = 0; i < N; ++i) cnt[i + 1] += cnt[i];
    int64_t* cand = malloc(sizeof(int64_t) * (size_t)(cnt[N] + 1));
    int64_t* cur = malloc(sizeof(int64_t) * (size_t)(N + 1));
    memcpy(cur, cnt, sizeof(int64_t) * (size_t)N);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) cand[cur[map[e * k + a]]++] = map[e * k + b];
    r->offsets = malloc(sizeof(int64_t) * (size_t)(N + 1));
    r->offsets[0] = 0;
    int64_t nnz = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t* row = &cand[cnt[i]];
        const int64_t len = cnt[i + 1] - cnt[i];
        qsort(row, (size_t)len, sizeof(int64_t), cmp_i64);
        int64_t u = 0;
        for (int64_t p = 0; p < len; ++p)
            if (u == 0 || row[p] != row[u - 1]) row[u++] = row[p];
        nnz += u;
        r->offsets[i + 1] = nnz;
        cur[i] = u;
    }
    r->nnz = nnz;
    r->cols = malloc(sizeof(int64_t) * (size_t)(nnz + 1));
    for (int64_t i = 0; i < N; ++i) memcpy(&r->cols[r->offsets[i]], &cand[cnt[i]], sizeof(int64_t) * (size_t)cur[i]);
    free(cand); free(cnt); free(cur);

    /* vector routing segments (routing.cpp:47-62) */
    r->vec_off = calloc((size_t)N + 1, sizeof(uint32_t));
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a) ++r->vec_off[map[e * k + a] + 1];
    for (int64_t i = 0; i < N; ++i) r->vec_off[i + 1] += r->vec_off[i];
    r->vec_slots = malloc(sizeof(uint32_t) * (size_t)(E * k + 1));
    uint32_t* c32 = malloc(sizeof(uint32_t) * (size_t)(nnz + N + 1));
    memcpy(c32, r->vec_off, sizeof(uint32_t) * (size_t)N);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a) r->vec_slots[c32[map[e * k + a]]++] = (uint32_t)(e * k + a);

    /* matrix routing segments (routing.cpp:64-83) */
    r->mat_off = calloc((size_t)nnz + 1, sizeof(uint32_t));
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) ++r->mat_off[find(r, map[e * k + a], map[e * k + b]) + 1];
    for (int64_t t = 0; t < nnz; ++t) r->mat_off[t + 1] += r->mat_off[t];
    r->mat_slots = malloc(sizeof(uint32_t) * (size_t)(E * k * k + 1));
    memcpy(c32, r->mat_off, sizeof(uint32_t) * (size_t)nnz);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) {
                const int64_t t = find(r, map[e * k + a], map[e * k + b]);
                r->mat_slots[c32[t]++] = (uint32_t)((e * k + a) * k + b);
            }
    free(c32);
    return r;
}

void tgo_routing_free(tgo_routing* r) {
    if (!r) return;
    free(r->offsets); free(r->cols); free(r->vec_off); free(r->vec_slots);
    free(r->mat_off); free(r->mat_slots); free(r);
}

int64_t tgo_routing_nnz(const tgo_routing* r) { return r->nnz; }

void tgo_routing_copy(const tgo_routing* r, int64_t* offsets, int64_t* cols, uint32_t* vec_off,
                      uint32_t* vec_slots, uint32_t* mat_off, uint32_t* mat_slots) {
    if (offsets) memcpy(offsets, r->offsets, sizeof(int64_t) * (size_t)(r->N + 1));
    if (cols) memcpy(cols, r->cols, sizeof(int64_t) * (size_t)r->nnz);
    if (vec_off) memcpy(vec_off, r->vec_off, sizeof(uint32_t) * (size_t)(r->N + 1));
    if (vec_slots) memcpy(vec_slots, r->vec_slots, sizeof(uint32_t) * (size_t)(r->E * r->k));
    if (mat_off) memcpy(mat_off, r->mat_off, sizeof(uint32_t) * (size_t)(r->nnz + 1));
    if (mat_slots) memcpy(mat_slots, r->mat_slots, sizeof(uint32_t) * (size_t)(r->E * r->k * r->k));
}

/* reduce_vector (routing.cpp:87-100) */
void tgo_reduce_vector(const tgo_routing* r, const double* local, double* F) {
    for (int64_t i = 0; i < r->N; ++i) {
        double s = 0.0;
        for (uint32_t t = r->vec_off[i]; t < r->vec_off[i + 1]; ++t) s += local[r->vec_slots[t]];
        F[i] = s;
    }
}

/* reduce_matrix (routing.cpp:109-125) */
void tgo_reduce_matrix(const tgo_routing* r, const double* local, double* values) {
    for (int64_t t = 0; t < r->nnz; ++t) {
        double s = 0.0;
        for (uint32_t u = r->mat_off[t]; u < r->mat_off[t + 1]; ++u) s += local[r->mat_slots[u]];
        values[t] = s;
    }
}

/* scatter_add_oracle (routing.cpp:163-174) */
void tgo_scatter_add(const tgo_routing* r, const int64_t* map, const double* localK,
                     const double* localF, double* values, double* F) {
    const int k = r->k;
    if (values) memset(values, 0, sizeof(double) * (size_t)r->nnz);
    if (F) memset(F, 0, sizeof(double) * (size_t)r->N);
    for (int64_t e = 0; e < r->E; ++e) {
        const int64_t* g = &map[e * k];
        if (localK && values) {
            const double* Ke = &localK[(size_t)e * k * k];
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) values[find(r, g[a], g[b])] += Ke[a * k + b];
        }
        if (localF && F) {
            const double* Fe = &localF[(size_t)e * k];
            for (int a = 0; a < k; ++a) F[g[a]] += Fe[a];
        }
    }
}

/* ------------------------------------------------------------------ assemble */

/* plane_stress_lambda (batch.cpp:359-361) */
static double plane_stress_lambda(double lambda, double mu) {
    return 2.0 * lambda * mu / (lambda + 2.0 * mu);
}

/* assemble (physics.cpp:10-75) */
int tgo_assemble(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                 int64_t n_elems, const tgo_routing* r, int problem, const tgo_field* diffusion,
                 const tgo_field* lambda, const tgo_field* mu, int plane_stress, int n_source,
                 const tgo_field* sources, int with_mass, double* K, double* F, double* M) {
    const int d = tgo_element_dim(kind), kg = tgo_element_nodes(kind);
    const int comps = problem == 1 ? d : 1;
    if (r->k != kg * comps)
        return fail(2, "assemble: dofmap component count does not match problem kind");
    const tgo_field one = {0, 1.0, NULL, 0};
    if (!diffusion) diffusion = &one;
    if (!lambda) lambda = &one;
    if (!mu) mu = &one;
    const int needs_high = diffusion->type != 0 || problem == 2 || with_mass;
    const int degree = tgo_default_degree(kind, needs_high);
    tables_t t;
    int rc = make_tables(kind, degree, &t);
    if (rc) return rc;
    geom_t g;
    rc = geometry(&t, nodes, elems, n_elems, &g, NULL);
    if (rc) return rc;
    const size_t nq = (size_t)n_elems * t.Q;
    const int k = r->k;
    double* c1 = malloc(sizeof(double) * nq * (size_t)d + 8);
    double* c2 = malloc(sizeof(double) * nq + 8);
    double* local = malloc(sizeof(double) * (size_t)n_elems * k * k + 8);
    int64_t* map = malloc(sizeof(int64_t) * (size_t)n_elems * k + 8);
    tgo_dofmap(kind, elems, n_elems, comps, map);
    (void)map;
    if (problem == 2) {
        if ((rc = evaluate(&t, elems, n_elems, n_nodes, diffusion, c1))) goto done;
        k_mass(&t, &g, c1, local);
        tgo_reduce_matrix(r, local, K);
        if (F) memset(F, 0, sizeof(double) * (size_t)r->N);
        goto done;
    }
    if (problem == 0) {
        if ((rc = evaluate(&t, elems, n_elems, n_nodes, diffusion, c1))) goto done;
        k_diffusion(&t, &g, c1, local);
        tgo_reduce_matrix(r, local, K);
        if (n_source > 0) {
            if ((rc = evaluate(&t, elems, n_elems, n_nodes, &sources[0], c1))) goto done;
            k_load(&t, &g, c1, local);
            tgo_reduce_vector(r, local, F);
        } else if (F) {
            memset(F, 0, sizeof(double) * (size_t)r->N);
        }
    } else {
        if ((rc = evaluate(&t, elems, n_elems, n_nodes, lambda, c1))) goto done;
        if ((rc = evaluate(&t, elems, n_elems, n_nodes, mu, c2))) goto done;
        if (d == 2 && plane_stress)
            for (size_t i = 0; i < nq; ++i) c1[i] = plane_stress_lambda(c1[i], c2[i]);
        if ((rc = k_elasticity(&t, &g, c1, c2, local))) goto done;
        tgo_reduce_matrix(r, local, K);
        if (n_source > 0) {
            if (n_source != d) {
                rc = fail(2, "elasticity body force needs one component per dimension");
                goto done;
            }
            double* comp = malloc(sizeof(double) * nq + 8);
            for (int c = 0; c < d; ++c) {
                if ((rc = evaluate(&t, elems, n_elems, n_nodes, &sources[c], comp))) {
                    free(comp);
                    goto done;
                }
                for (size_t i = 0; i < nq; ++i) c1[i * d + c] = comp[i];
            }
            free(comp);
            k_load_vector(&t, &g, c1, local);
            tgo_reduce_vector(r, local, F);
        } else if (F) {
            memset(F, 0, sizeof(double) * (size_t)r->N);
        }
    }
    if (with_mass) {
        if (comps != 1) {
            rc = fail(2, "mass matrix assembly only supported for scalar fields");
            goto done;
        }
        for (size_t i = 0; i < nq; ++i) c1[i] = 1.0;
        k_mass(&t, &g, c1, local);
        tgo_reduce_matrix(r, local, M);
    }
done:
    free(c1); free(c2); free(local); free(map);
    geom_free(&g);
    return rc;
}

/* gradient_products (adjoint.cpp:68-82) */
void tgo_gradient_products(const tgo_routing* r, const double* lambda, const double* U,
                           double* dK, double* dF) {
    for (int64_t i = 0; i < r->N; ++i)
        for (int64_t t = r->offsets[i]; t < r->offsets[i + 1]; ++t) dK[t] = lambda[i] * U[r->cols[t]];
    if (dF)
        for (int64_t i = 0; i < r->N; ++i) dF[i] = -lambda[i];
}

/* tg_main.cpp:846-850: grad += lam[map[a]] * K_unit[(e*k+a)*k+b] * U[map[b]] */
void tgo_adjoint_gather(int64_t E, int k, const int64_t* map, const double* K0,
                        const double* lambda, const double* U, double* out) {
    for (int64_t e = 0; e < E; ++e) {
        const int64_t* g = &map[e * k];
        double grad = 0.0;
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) grad += lambda[g[a]] * K0[((size_t)e * k + a) * k + b] * U[g[b]];
        out[e] = grad;
    }
}

/* acceptance.cpp:372-377 with the sign flipped (out = -generic) */
void tgo_adjoint_generic(const tgo_routing* r, const int64_t* map, const double* K0,
                         const double* dK, double* out) {
    const int k = r->k;
    for (int64_t e = 0; e < r->E; ++e) {
        const int64_t* g = &map[e * k];
        double s = 0.0;
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) s += dK[find(r, g[a], g[b])] * K0[((size_t)e * k + a) * k + b];
        out[e] = s;
    }
}
