// Host half of libtgk.so: error state, the reference-compatible mesh helpers
// (grid generation, content hash, boundary, validation, quadrature tables),
// device mesh handles, the fused-plan upload and the tg::assemble dispatcher.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <type_traits>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <climits>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "tgk_internal.hpp"

namespace tgk {

namespace {
thread_local std::string g_err;
std::atomic<int> g_threads{0};
}  // namespace

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
const std::string& last_error() { return g_err; }

#define HCUDA(call)                                                                    \
    do {                                                                               \
        cudaError_t _e = (call);                                                       \
        if (_e != cudaSuccess)                                                         \
            return set_error(TGK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

static int host_ensure_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return set_error(TGK_ERR_CUDA, "no usable CUDA device (libtgk has no CPU fallback)");
    return TGK_OK;
}

// ---------------------------------------------------------------- reference tables
// reference.cpp:45-71 (shape functions) and :99-210 (rules), host copy.
static void shape_values(int kind, const double* p, double* v) {
    if (kind == TGK_TRI3) {
        v[0] = 1.0 - p[0] - p[1]; v[1] = p[0]; v[2] = p[1];
    } else if (kind == TGK_QUAD4) {
        const double x = p[0], y = p[1];
        v[0] = (1 - x) * (1 - y); v[1] = x * (1 - y); v[2] = x * y; v[3] = (1 - x) * y;
    } else {
        v[0] = 1.0 - p[0] - p[1] - p[2]; v[1] = p[0]; v[2] = p[1]; v[3] = p[2];
    }
}

static void shape_gradients(int kind, const double* p, double* g) {
    if (kind == TGK_TRI3) {
        const double t[6] = {-1, -1, 1, 0, 0, 1};
        std::memcpy(g, t, sizeof t);
    } else if (kind == TGK_QUAD4) {
        const double x = p[0], y = p[1];
        const double t[8] = {-(1 - y), -(1 - x), (1 - y), -x, y, x, -y, (1 - x)};
        std::memcpy(g, t, sizeof t);
    } else {
        const double t[12] = {-1, -1, -1, 1, 0, 0, 0, 1, 0, 0, 0, 1};
        std::memcpy(g, t, sizeof t);
    }
}

static int rule(int kind, int degree, int& Q, std::vector<double>& pts, std::vector<double>& w) {
    if (degree < 1 || degree > 4)
        return set_error(TGK_ERR_INPUT, "quadrature degree " + std::to_string(degree) +
                                            " unsupported; supported degrees: 1,2,3,4");
    if (kind == TGK_TRI3) {
        switch (degree) {
            case 1: Q = 1; pts = {1.0 / 3.0, 1.0 / 3.0}; w = {0.5}; break;
            case 2: Q = 3; pts = {1.0 / 6, 1.0 / 6, 2.0 / 3, 1.0 / 6, 1.0 / 6, 2.0 / 3};
                    w = {1.0 / 6, 1.0 / 6, 1.0 / 6}; break;
            case 3: Q = 4; pts = {1.0 / 3, 1.0 / 3, 0.2, 0.2, 0.6, 0.2, 0.2, 0.6};
                    w = {-27.0 / 96, 25.0 / 96, 25.0 / 96, 25.0 / 96}; break;
            default: {
                const double a1 = 0.445948490915965, w1 = 0.223381589678011;
                const double a2 = 0.091576213509771, w2 = 0.109951743655322;
                Q = 6;
                pts = {a1, a1, 1 - 2 * a1, a1, a1, 1 - 2 * a1, a2, a2, 1 - 2 * a2, a2, a2, 1 - 2 * a2};
                w = {w1 / 2, w1 / 2, w1 / 2, w2 / 2, w2 / 2, w2 / 2};
            }
        }
    } else if (kind == TGK_QUAD4) {
        std::vector<double> g, gw;
        if (degree <= 1) { g = {0.5}; gw = {1.0}; }
        else if (degree <= 3) { const double s = 0.5 / std::sqrt(3.0); g = {0.5 - s, 0.5 + s}; gw = {0.5, 0.5}; }
        else { const double s = 0.5 * std::sqrt(0.6); g = {0.5 - s, 0.5, 0.5 + s}; gw = {5.0 / 18, 8.0 / 18, 5.0 / 18}; }
        const int n = static_cast<int>(g.size());
        Q = n * n;
        pts.clear(); w.clear();
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) { pts.push_back(g[i]); pts.push_back(g[j]); w.push_back(gw[i] * gw[j]); }
    } else {
        switch (degree) {
            case 1: Q = 1; pts = {0.25, 0.25, 0.25}; w = {1.0 / 6.0}; break;
            case 2: {
                const double a = 0.585410196624969, b = 0.138196601125011;
                Q = 4; pts = {b, b, b, a, b, b, b, a, b, b, b, a}; w.assign(4, 1.0 / 24.0); break;
            }
            case 3: {
                const double s = 1.0 / 6.0;
                Q = 5; pts = {0.25, 0.25, 0.25, s, s, s, 0.5, s, s, s, 0.5, s, s, s, 0.5};
                w = {-4.0 / 5.0 / 6.0, 9.0 / 20.0 / 6.0, 9.0 / 20.0 / 6.0, 9.0 / 20.0 / 6.0, 9.0 / 20.0 / 6.0};
                break;
            }
            default: {
                const double a = 11.0 / 14.0, b = 1.0 / 14.0;
                const double c = 0.399403576166799, dd = 0.100596423833201;
                const double w1 = -74.0 / 5625.0, w2 = 343.0 / 45000.0, w3 = 56.0 / 2250.0;
                Q = 11;
                pts = {0.25, 0.25, 0.25, b, b, b, a, b, b, b, a, b, b, b, a,
                       c, dd, dd, dd, c, dd, dd, dd, c, dd, c, c, c, dd, c, c, c, dd};
                w = {w1, w2, w2, w2, w2, w3, w3, w3, w3, w3, w3};
            }
        }
    }
    return TGK_OK;
}

// centroid_det (mesh.cpp:31-52)
static double centroid_det(int kind, const double* nodes, const int64_t* conn) {
    const int k = element_nodes(kind), d = element_dim(kind);
    static const double ref_nodes[3][4][3] = {{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 0}},
                                              {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}},
                                              {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
    double centroid[3] = {0, 0, 0};
    for (int a = 0; a < k; ++a)
        for (int c = 0; c < d; ++c) centroid[c] += ref_nodes[kind][a][c] / k;
    double g[12];
    shape_gradients(kind, centroid, g);
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
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

int narrow_connectivity_async(tgk_mesh* m, const int64_t* src, int64_t n, int64_t n_nodes, int32_t* dst,
                              cudaStream_t st);
int mesh_async_flags(tgk_mesh* m, int64_t* bad, bool* changed);
int narrow_connectivity(tgk_mesh* m, const int64_t* src, int64_t n, int64_t n_nodes, int32_t* dst, int64_t* bad,
                        cudaStream_t st);
int fused_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                          double* F, double* M, cudaStream_t st, unsigned long long* d_bad);
int fast_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F, double* M,
                         cudaStream_t st, unsigned long long* d_bad);
int materialised_scalar_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                                 double* M, cudaStream_t st, unsigned long long* d_bad);
int fast_elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                             cudaStream_t st);
int elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K,
                        double* F, cudaStream_t st);
int fused_elasticity_assemble(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                              cudaStream_t st);
int fused_allen_cahn(const tgk_mesh* m, tgk_routing* r, const double* u, double eps, double* T, double* F,
                     cudaStream_t st);
int fused_scalar_assemble_f32(const tgk_problem* pr, const tgk_mesh* m, tgk_routing* r, float* K, float* F,
                              float* M, cudaStream_t st, unsigned long long* d_bad);

}  // namespace tgk

using namespace tgk;

extern "C" {

const char* tgk_last_error(void) { return last_error().c_str(); }
int tgk_version(void) { return 1; }
int tgk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}
void tgk_set_thread_count(int n) { g_threads.store(n < 0 ? 0 : n); }
int tgk_thread_count(void) {
    int n = g_threads.load();
    if (n == 0) n = std::max(1u, std::thread::hardware_concurrency());
    return n;
}

int tgk_default_degree(int kind, int mass) {
    if (kind == TGK_QUAD4) return 3;
    return mass ? 2 : 1;
}

int tgk_tables(int kind, int degree, int* Q, double* points, double* weights, double* B, double* G) {
    int q;
    std::vector<double> pts, w;
    TGK_TRY(rule(kind, degree, q, pts, w));
    const int k = element_nodes(kind), d = element_dim(kind);
    *Q = q;
    if (points) std::memcpy(points, pts.data(), sizeof(double) * q * d);
    if (weights) std::memcpy(weights, w.data(), sizeof(double) * q);
    for (int i = 0; i < q; ++i) {
        double v[4], g[12];
        shape_values(kind, &pts[i * d], v);
        shape_gradients(kind, &pts[i * d], g);
        for (int a = 0; a < k; ++a) {
            if (B) B[i * k + a] = v[a];
            for (int c = 0; c < d; ++c)
                if (G) G[(i * k + a) * d + c] = g[a * d + c];
        }
    }
    return TGK_OK;
}

int tgk_grid_sizes(int kind, const int64_t* div, int64_t* n_nodes, int64_t* n_elems) {
    const int d = element_dim(kind);
    for (int c = 0; c < d; ++c)
        if (div[c] < 1) return set_error(TGK_ERR_INPUT, "generate_grid: divisions must be >= 1");
    if (d == 3) {
        *n_nodes = (div[0] + 1) * (div[1] + 1) * (div[2] + 1);
        *n_elems = 6 * div[0] * div[1] * div[2];
    } else {
        *n_nodes = (div[0] + 1) * (div[1] + 1);
        *n_elems = (kind == TGK_TRI3 ? 2 : 1) * div[0] * div[1];
    }
    return TGK_OK;
}

// generate_grid (mesh.cpp:96-169), same node order, Kuhn permutations and
// orientation fix; threaded over z for large grids.
int tgk_generate_grid(int kind, const double* ext, const int64_t* div, double* nodes, int64_t* elems) {
    int64_t nn, ne;
    TGK_TRY(tgk_grid_sizes(kind, div, &nn, &ne));
    if (!nodes || !elems) return TGK_OK;
    if (element_dim(kind) == 2) {
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
                if (kind == TGK_QUAD4) {
                    elems[q++] = n00; elems[q++] = n10; elems[q++] = n11; elems[q++] = n01;
                } else {
                    elems[q++] = n00; elems[q++] = n10; elems[q++] = n11;
                    elems[q++] = n00; elems[q++] = n11; elems[q++] = n01;
                }
            }
        return TGK_OK;
    }
    const int64_t nx = div[0], ny = div[1], nz = div[2];
    const double hx = ext[0] / nx, hy = ext[1] / ny, hz = ext[2] / nz;
    auto node_work = [&](int64_t z0, int64_t z1) {
        for (int64_t kz = z0; kz < z1; ++kz)
            for (int64_t j = 0; j <= ny; ++j)
                for (int64_t i = 0; i <= nx; ++i) {
                    const int64_t p = 3 * (i + (nx + 1) * (j + (ny + 1) * kz));
                    nodes[p] = i * hx;
                    nodes[p + 1] = j * hy;
                    nodes[p + 2] = kz * hz;
                }
    };
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    auto elem_work = [&](int64_t z0, int64_t z1) {
        for (int64_t kz = z0; kz < z1; ++kz)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t i = 0; i < nx; ++i)
                    for (int s6 = 0; s6 < 6; ++s6) {
                        const int64_t e = ((kz * ny + j) * nx + i) * 6 + s6;
                        int64_t* tet = &elems[e * 4];
                        int64_t c[3] = {0, 0, 0};
                        tet[0] = i + (nx + 1) * (j + (ny + 1) * kz);
                        for (int s = 0; s < 3; ++s) {
                            c[perms[s6][s]] = 1;
                            tet[s + 1] = (i + c[0]) + (nx + 1) * ((j + c[1]) + (ny + 1) * (kz + c[2]));
                        }
                        if (centroid_det(kind, nodes, tet) < 0.0) std::swap(tet[2], tet[3]);
                    }
    };
    const int nt = std::max(1, std::min<int>(tgk_thread_count(), 32));
    auto par = [&](auto fn, int64_t n) {
        std::vector<std::thread> pool;
        const int64_t per = (n + nt - 1) / nt;
        for (int t = 0; t < nt; ++t) {
            const int64_t a = t * per, b = std::min(n, a + per);
            if (a < b) pool.emplace_back(fn, a, b);
        }
        for (auto& th : pool) th.join();
    };
    par(node_work, nz + 1);
    par(elem_work, nz);
    return TGK_OK;
}

// Mesh::content_hash (mesh.cpp:79-94), FNV-1a
uint64_t tgk_content_hash(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                          int64_t n_elems) {
    uint64_t h = 14695981039346656037ull;
    auto mix = [&h](const void* data, size_t n) {
        const auto* p = static_cast<const unsigned char*>(data);
        for (size_t i = 0; i < n; ++i) {
            h ^= p[i];
            h *= 1099511628211ull;
        }
    };
    const int kind_tag = kind, dim = element_dim(kind);
    mix(&kind_tag, sizeof kind_tag);
    mix(&dim, sizeof dim);
    mix(nodes, static_cast<size_t>(n_nodes) * dim * sizeof(double));
    mix(elems, static_cast<size_t>(n_elems) * element_nodes(kind) * sizeof(int64_t));
    return h;
}

// topological_boundary (mesh.cpp:185-209): nodes of facets owned by one element
int64_t tgk_topological_boundary(int kind, const int64_t* elems, int64_t n_elems, int64_t n_nodes,
                                 int64_t* out) {
    const int k = element_nodes(kind);
    std::vector<std::vector<int>> facets;
    switch (kind) {
        case TGK_TRI3: facets = {{0, 1}, {1, 2}, {2, 0}}; break;
        case TGK_QUAD4: facets = {{0, 1}, {1, 2}, {2, 3}, {3, 0}}; break;
        default: facets = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}}; break;
    }
    const int fs = static_cast<int>(facets[0].size());
    std::vector<std::array<int64_t, 3>> keys;
    keys.reserve(static_cast<size_t>(n_elems) * facets.size());
    for (int64_t e = 0; e < n_elems; ++e)
        for (const auto& f : facets) {
            std::array<int64_t, 3> key{-1, -1, -1};
            for (int i = 0; i < fs; ++i) key[i] = elems[e * k + f[i]];
            std::sort(key.begin(), key.begin() + fs);
            keys.push_back(key);
        }
    std::sort(keys.begin(), keys.end());
    std::vector<char> on(static_cast<size_t>(n_nodes), 0);
    for (size_t i = 0; i < keys.size();) {
        size_t j = i;
        while (j < keys.size() && keys[j] == keys[i]) ++j;
        if (j - i == 1)
            for (int c = 0; c < fs; ++c) on[keys[i][c]] = 1;
        i = j;
    }
    int64_t n = 0;
    for (int64_t v = 0; v < n_nodes; ++v)
        if (on[v]) {
            if (out) out[n] = v;
            ++n;
        }
    return n;
}

// Mesh::validate (mesh.cpp:56-77)
int tgk_validate(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems, int64_t n_elems) {
    const int k = element_nodes(kind);
    for (int64_t e = 0; e < n_elems; ++e) {
        const int64_t* conn = &elems[e * k];
        for (int a = 0; a < k; ++a) {
            if (conn[a] < 0 || conn[a] >= n_nodes)
                return set_error(TGK_ERR_INPUT, "element " + std::to_string(e) + " references node " +
                                                    std::to_string(conn[a]) + " outside [0," +
                                                    std::to_string(n_nodes) + ")");
            for (int b = a + 1; b < k; ++b)
                if (conn[a] == conn[b])
                    return set_error(TGK_ERR_INPUT, "element " + std::to_string(e) + " repeats node " +
                                                        std::to_string(conn[a]));
        }
        if (centroid_det(kind, nodes, conn) <= 0.0)
            return set_error(TGK_ERR_INPUT, "element " + std::to_string(e) +
                                                " has non-positive orientation (det J <= 0)");
    }
    return TGK_OK;
}

// ---------------------------------------------------------------- mesh handles
int tgk_mesh_create(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                    int64_t n_elems, tgk_mesh** out) {
    if (!out) return set_error(TGK_ERR_INPUT, "tgk_mesh_create: null out");
    if (kind != TGK_TRI3 && kind != TGK_TET4 && kind != TGK_QUAD4)
        return set_error(TGK_ERR_INPUT, "unknown element kind");
    if (n_nodes > INT32_MAX) return set_error(TGK_ERR_INPUT, "mesh has more than 2^31-1 nodes");
    TGK_TRY(host_ensure_device());
    auto* m = new tgk_mesh();
    m->kind = kind;
    m->d = element_dim(kind);
    m->k = element_nodes(kind);
    m->N = n_nodes;
    m->E = n_elems;
    m->owned = true;
    if (cudaMalloc(&m->nodes, sizeof(double) * std::max<int64_t>(1, n_nodes * m->d)) != cudaSuccess ||
        cudaMalloc(&m->conn, sizeof(int32_t) * std::max<int64_t>(1, n_elems * m->k)) != cudaSuccess) {
        tgk_mesh_destroy(m);
        return set_error(TGK_ERR_CUDA, "tgk_mesh_create: cudaMalloc failed");
    }
    int rc = tgk_mesh_upload(m, nodes, elems, nullptr);
    if (rc != TGK_OK) {
        tgk_mesh_destroy(m);
        return rc;
    }
    *out = m;
    return TGK_OK;
}

int tgk_mesh_create_d(int kind, const double* d_nodes, int64_t n_nodes, const int32_t* d_elems,
                      int64_t n_elems, tgk_mesh** out) {
    if (!out) return set_error(TGK_ERR_INPUT, "tgk_mesh_create_d: null out");
    auto* m = new tgk_mesh();
    m->kind = kind;
    m->d = element_dim(kind);
    m->k = element_nodes(kind);
    m->N = n_nodes;
    m->E = n_elems;
    m->nodes = const_cast<double*>(d_nodes);
    m->conn = const_cast<int32_t*>(d_elems);
    m->owned = false;
    *out = m;
    return TGK_OK;
}

int tgk_mesh_upload(tgk_mesh* m, const double* nodes, const int64_t* elems, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nodes) {
        HCUDA(cudaMemcpyAsync(m->nodes, nodes, sizeof(double) * m->N * m->d, cudaMemcpyHostToDevice, st));
        m->div_safe = -1;  // re-certified lazily by the fused path
    }
    if (elems) {
        // int64 connectivity goes over PCIe as is and is narrowed (and range
        // checked, mesh.cpp:61-64) by a device kernel
        const int64_t n = m->E * m->k;
        if (!m->staging) HCUDA(cudaMalloc(&m->staging, sizeof(int64_t) * std::max<int64_t>(1, n)));
        HCUDA(cudaMemcpyAsync(m->staging, elems, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        int64_t bad = -1;
        TGK_TRY(narrow_connectivity(m, m->staging, n, m->N, m->conn, &bad, st));
        if (bad >= 0)
            return set_error(TGK_ERR_INPUT, "element " + std::to_string(bad / m->k) + " references node " +
                                                std::to_string(elems[bad]) + " outside [0," +
                                                std::to_string(m->N) + ")");
    } else {
        HCUDA(cudaStreamSynchronize(st));
    }
    return TGK_OK;
}

// Stream-ordered variant for pipelined callers: no host synchronisation; the
// connectivity range check and change detection accumulate on the device
// until tgk_mesh_upload_check.
int tgk_mesh_upload_async(tgk_mesh* m, const double* nodes, const int64_t* elems, void* stream) {
    if (!m) return set_error(TGK_ERR_INPUT, "null mesh");
    if (!m->owned) return set_error(TGK_ERR_INPUT, "tgk_mesh_upload_async: wrapped (tgk_mesh_create_d) mesh");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nodes) {
        HCUDA(cudaMemcpyAsync(m->nodes, nodes, sizeof(double) * m->N * m->d, cudaMemcpyHostToDevice, st));
        m->div_safe = -1;
    }
    if (elems) {
        const int64_t n = m->E * m->k;
        if (!m->staging) HCUDA(cudaMalloc(&m->staging, sizeof(int64_t) * std::max<int64_t>(1, n)));
        HCUDA(cudaMemcpyAsync(m->staging, elems, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        TGK_TRY(narrow_connectivity_async(m, m->staging, n, m->N, m->conn, st));
    }
    return TGK_OK;
}

int tgk_mesh_upload_check(tgk_mesh* m) {
    if (!m) return set_error(TGK_ERR_INPUT, "null mesh");
    int64_t bad = -1;
    bool changed = false;
    TGK_TRY(mesh_async_flags(m, &bad, &changed));
    if (changed) ++m->conn_version;  // routings built before refuse to assemble (check_routing_fresh)
    if (bad >= 0)
        return set_error(TGK_ERR_INPUT, "element " + std::to_string(bad / m->k) + " references a node outside [0," +
                                            std::to_string(m->N) + ")");
    return TGK_OK;
}

int tgk_mesh_coordinates_changed(tgk_mesh* m) {
    if (!m) return set_error(TGK_ERR_INPUT, "null mesh");
    m->div_safe = -1;  // re-certified for the Markstein division on the next fused call
    return TGK_OK;
}

void tgk_mesh_destroy(tgk_mesh* m) {
    if (!m) return;
    if (m->owned) {
        if (m->nodes) cudaFree(m->nodes);
        if (m->conn) cudaFree(m->conn);
    }
    if (m->staging) cudaFree(m->staging);
    if (m->d_flags) cudaFree(m->d_flags);
    if (m->h_flags) cudaFreeHost(m->h_flags);
    delete m;
}

int tgk_mesh_info(const tgk_mesh* m, int* kind, int64_t* n_nodes, int64_t* n_elems,
                  const double** d_nodes, const int32_t** d_elems) {
    if (!m) return set_error(TGK_ERR_INPUT, "null mesh");
    if (kind) *kind = m->kind;
    if (n_nodes) *n_nodes = m->N;
    if (n_elems) *n_elems = m->E;
    if (d_nodes) *d_nodes = m->nodes;
    if (d_elems) *d_elems = m->conn;
    return TGK_OK;
}

// Restrict the fused assembly to the owned scalar rows [lo, hi) (row-owning
// partitions); other rows of the outputs are left untouched.
int tgk_routing_set_owned_rows(tgk_routing* r, int64_t lo, int64_t hi) {
    tgk_routing* s = r->scalar ? r->scalar : r;
    if (lo < 0 || hi > s->N || lo > hi) return set_error(TGK_ERR_INPUT, "owned row range out of bounds");
    if (s->own_lo == lo && s->own_hi == hi) return TGK_OK;
    for (auto& pl : s->plan) pl.release();
    s->entry_plan.release();
    for (auto& fp : s->fast_plan) fp.release();
    s->fast_plan_used = nullptr;
    s->own_lo = lo;
    s->own_hi = hi;
    return TGK_OK;
}

// Restrict the fused assembly to the elements [lo, hi) (multi-GPU slabs that
// exchange interface partial sums): rows touched only by other elements get
// +0.0, rows shared with other elements get the partial fold of these.
int tgk_routing_set_element_range(tgk_routing* r, int64_t lo, int64_t hi) {
    tgk_routing* s = r->scalar ? r->scalar : r;
    if (lo < 0 || hi > s->E || lo > hi) return set_error(TGK_ERR_INPUT, "element range out of bounds");
    if (s->elem_lo == lo && s->elem_hi == hi) return TGK_OK;
    for (auto& pl : s->plan) pl.release();
    for (auto& fp : s->fast_plan) fp.release();
    s->fast_plan_used = nullptr;
    s->elem_lo = lo;
    s->elem_hi = hi;
    return TGK_OK;
}

// Plan statistics: blocks, halo elements (recompute factor = halo / E), records, bytes.
int tgk_routing_plan_stats(tgk_routing* r, int rows_per_block, int64_t* n_blocks, int64_t* n_halo,
                           int64_t* n_records, int64_t* bytes) {
    const PlanDev* pl = nullptr;
    TGK_TRY(ensure_plan(r, rows_per_block == 128 || rows_per_block == 64 ? rows_per_block : 256, &pl));
    if (n_blocks) *n_blocks = pl->n_blocks;
    if (n_halo) *n_halo = pl->n_halo;
    if (n_records) *n_records = pl->n_records;
    if (bytes) *bytes = pl->bytes;
    return TGK_OK;
}

// routing cache in the reference layout (routing.cpp:178-209)
int tgk_routing_save(const tgk_routing* r, uint64_t mesh_hash, const char* path) {
    if (!r->mat_offsets || !r->vec_offsets)
        return set_error(TGK_ERR_INPUT, "tgk_routing_save: routing built without TGK_ROUTING_SEGMENTS");
    const size_t Ek = static_cast<size_t>(r->E) * r->k;
    std::vector<int64_t> off(r->N + 1), cols(r->nnz);
    std::vector<uint32_t> vo(r->N + 1), vs(Ek), mo(r->nnz + 1), ms(Ek * r->k);
    TGK_TRY(tgk_routing_copy(r, off.data(), cols.data(), nullptr, vo.data(), vs.data(), mo.data(), ms.data()));
    FILE* f = std::fopen(path, "wb");
    if (!f) return set_error(TGK_ERR_INPUT, std::string("cannot open routing cache for writing: ") + path);
    const int64_t header[6] = {static_cast<int64_t>(0x74672d726f757432ull), static_cast<int64_t>(mesh_hash),
                               r->N, r->E, r->k, r->nnz};
    std::fwrite(header, sizeof header, 1, f);
    std::fwrite(off.data(), 8, off.size(), f);
    std::fwrite(cols.data(), 8, cols.size(), f);
    std::fwrite(vo.data(), 4, vo.size(), f);
    std::fwrite(vs.data(), 4, vs.size(), f);
    std::fwrite(mo.data(), 4, mo.size(), f);
    std::fwrite(ms.data(), 4, ms.size(), f);
    std::fclose(f);
    return TGK_OK;
}

}  // extern "C"

namespace tgk {

void PlanDev::release() {
    for (void* p : {(void*)row_off, (void*)rows, (void*)rows_rp, (void*)halo_off, (void*)halo, (void*)bnode_off,
                    (void*)bnodes, (void*)halo_lconn,
                    (void*)chunk_off, (void*)chunk_rec_off, (void*)chunk_row_off, (void*)recs})
        if (p) cudaFree(p);
    *this = PlanDev{};
}

// Host copies of the mesh and the scalar routing arrays the plans are built from.
int fetch_scalar_routing(const tgk_routing* r, ScalarRoutingHost& h) {
    const tgk_mesh* m = r->mesh;
    const int k = m->k, d = m->d;
    h.nodes.resize(m->N * d);
    h.conn.resize(m->E * k);
    h.row_ptr.resize(r->N + 1);
    h.vo.resize(r->N + 1);
    h.vs.resize(r->E * k);
    h.slot.resize(r->E * k * k);
    HCUDA(cudaMemcpy(h.nodes.data(), m->nodes, h.nodes.size() * 8, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(h.conn.data(), m->conn, h.conn.size() * 4, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(h.row_ptr.data(), r->row_ptr, h.row_ptr.size() * 8, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(h.vo.data(), r->vec_offsets, h.vo.size() * 4, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(h.vs.data(), r->vec_slots, h.vs.size() * 4, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(h.slot.data(), r->slot_of, h.slot.size() * 4, cudaMemcpyDeviceToHost));
    return TGK_OK;
}

void EntryPlanDev::release() {
    if (blob) cudaFree(blob);
    *this = EntryPlanDev{};
}

// Build (once per R and owned row range) and upload the batched kernel's entry plan.
int ensure_entry_plan(tgk_routing* rr, int R, const EntryPlanDev** out) {
    tgk_routing* r = rr->scalar ? rr->scalar : rr;
    EntryPlanDev& D = r->entry_plan;
    if (D.blob && D.R == R) {
        *out = &D;
        return TGK_OK;
    }
    D.release();
    const tgk_mesh* m = r->mesh;
    ScalarRoutingHost h;
    TGK_TRY(fetch_scalar_routing(r, h));
    EntryPlanHost P;
    const int64_t lo = r->own_hi < 0 ? 0 : r->own_lo, hi = r->own_hi < 0 ? r->N : r->own_hi;
    TGK_TRY(build_entry_plan(m->kind, m->N, h.nodes.data(), h.conn.data(), h.row_ptr.data(), h.vo.data(),
                             h.vs.data(), h.slot.data(), lo, hi, R, P));
    // one allocation, 16-byte aligned segments
    size_t total = 0;
    auto reserve = [&total](const auto& v) {
        const size_t at = total;
        total += (v.size() * sizeof(v[0]) + 15) & ~size_t(15);
        return at;
    };
    const size_t o_row_off = reserve(P.row_off), o_halo_off = reserve(P.halo_off), o_bnode_off = reserve(P.bnode_off),
                 o_ent_off = reserve(P.ent_off), o_contrib_off = reserve(P.contrib_off),
                 o_fcontrib_off = reserve(P.fcontrib_off), o_epos = reserve(P.epos), o_epos2 = reserve(P.epos2), o_rows = reserve(P.rows),
                 o_halo = reserve(P.halo), o_bnodes = reserve(P.bnodes), o_contrib = reserve(P.contrib),
                 o_fcontrib = reserve(P.fcontrib), o_coff = reserve(P.coff), o_fcoff = reserve(P.fcoff),
                 o_hconn = reserve(P.hconn);
    std::vector<unsigned char> img(std::max<size_t>(total, 16));
    auto put = [&img](size_t at, const auto& v) {
        if (!v.empty()) std::memcpy(img.data() + at, v.data(), v.size() * sizeof(v[0]));
    };
    put(o_row_off, P.row_off); put(o_halo_off, P.halo_off); put(o_bnode_off, P.bnode_off);
    put(o_ent_off, P.ent_off); put(o_contrib_off, P.contrib_off); put(o_fcontrib_off, P.fcontrib_off);
    put(o_epos, P.epos); put(o_epos2, P.epos2); put(o_rows, P.rows); put(o_halo, P.halo); put(o_bnodes, P.bnodes);
    put(o_contrib, P.contrib); put(o_fcontrib, P.fcontrib); put(o_coff, P.coff); put(o_fcoff, P.fcoff);
    put(o_hconn, P.hconn);
    void* blob = nullptr;
    HCUDA(cudaMalloc(&blob, img.size()));
    const cudaError_t ce = cudaMemcpy(blob, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        cudaFree(blob);
        return set_error(TGK_ERR_CUDA, std::string("entry plan upload: ") + cudaGetErrorString(ce));
    }
    auto* base = static_cast<unsigned char*>(blob);
    D.blob = blob;
    D.bytes = static_cast<int64_t>(img.size());
    D.R = R;
    D.n_blocks = P.n_blocks;
    D.max_halo = P.max_halo;
    D.max_bnodes = P.max_bnodes;
    D.max_contrib = P.max_contrib;
    D.max_fcontrib = P.max_fcontrib;
    D.max_entries = P.max_entries;
    D.max_clen = P.max_clen;
    D.row_off = reinterpret_cast<const int64_t*>(base + o_row_off);
    D.halo_off = reinterpret_cast<const int64_t*>(base + o_halo_off);
    D.bnode_off = reinterpret_cast<const int64_t*>(base + o_bnode_off);
    D.ent_off = reinterpret_cast<const int64_t*>(base + o_ent_off);
    D.contrib_off = reinterpret_cast<const int64_t*>(base + o_contrib_off);
    D.fcontrib_off = reinterpret_cast<const int64_t*>(base + o_fcontrib_off);
    D.epos = reinterpret_cast<const int64_t*>(base + o_epos);
    D.epos2 = reinterpret_cast<const int64_t*>(base + o_epos2);
    D.rows = reinterpret_cast<const uint32_t*>(base + o_rows);
    D.halo = reinterpret_cast<const uint32_t*>(base + o_halo);
    D.bnodes = reinterpret_cast<const uint32_t*>(base + o_bnodes);
    D.contrib = reinterpret_cast<const uint32_t*>(base + o_contrib);
    D.fcontrib = reinterpret_cast<const uint32_t*>(base + o_fcontrib);
    D.coff = reinterpret_cast<const uint32_t*>(base + o_coff);
    D.fcoff = reinterpret_cast<const uint32_t*>(base + o_fcoff);
    D.hconn = reinterpret_cast<const uint64_t*>(base + o_hconn);
    *out = &D;
    return TGK_OK;
}

void GroupPlanDev::release() {
    if (blob) cudaFree(blob);
    *this = GroupPlanDev{};
}

// Build (once per group size) and upload the adjoint gather's element-group plan.
int ensure_group_plan(tgk_routing* rr, int G, const GroupPlanDev** out) {
    tgk_routing* r = rr->scalar ? rr->scalar : rr;
    GroupPlanDev& D = r->group_plan;
    if (D.blob && D.G == G) {
        *out = &D;
        return TGK_OK;
    }
    D.release();
    const tgk_mesh* m = r->mesh;
    std::vector<double> nodes(m->N * m->d);
    std::vector<int32_t> conn(m->E * m->k);
    HCUDA(cudaMemcpy(nodes.data(), m->nodes, nodes.size() * 8, cudaMemcpyDeviceToHost));
    HCUDA(cudaMemcpy(conn.data(), m->conn, conn.size() * 4, cudaMemcpyDeviceToHost));
    GroupPlanHost P;
    TGK_TRY(build_group_plan(m->kind, m->N, m->E, nodes.data(), conn.data(), G, P));
    size_t total = 0;
    auto reserve = [&total](const auto& v) {
        const size_t at = total;
        total += (v.size() * sizeof(v[0]) + 15) & ~size_t(15);
        return at;
    };
    const size_t o_grp = reserve(P.grp_off), o_node = reserve(P.node_off), o_el = reserve(P.elems),
                 o_gn = reserve(P.gnodes), o_lc = reserve(P.lconn);
    std::vector<unsigned char> img(std::max<size_t>(total, 16));
    auto put = [&img](size_t at, const auto& v) {
        if (!v.empty()) std::memcpy(img.data() + at, v.data(), v.size() * sizeof(v[0]));
    };
    put(o_grp, P.grp_off); put(o_node, P.node_off); put(o_el, P.elems); put(o_gn, P.gnodes); put(o_lc, P.lconn);
    void* blob = nullptr;
    HCUDA(cudaMalloc(&blob, img.size()));
    const cudaError_t ce = cudaMemcpy(blob, img.data(), img.size(), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        cudaFree(blob);
        return set_error(TGK_ERR_CUDA, std::string("group plan upload: ") + cudaGetErrorString(ce));
    }
    auto* base = static_cast<unsigned char*>(blob);
    D.blob = blob;
    D.bytes = static_cast<int64_t>(img.size());
    D.G = G;
    D.n_groups = P.n_groups;
    D.max_nodes = P.max_nodes;
    D.grp_off = reinterpret_cast<const int64_t*>(base + o_grp);
    D.node_off = reinterpret_cast<const int64_t*>(base + o_node);
    D.elems = reinterpret_cast<const uint32_t*>(base + o_el);
    D.gnodes = reinterpret_cast<const uint32_t*>(base + o_gn);
    D.lconn = reinterpret_cast<const uint64_t*>(base + o_lc);
    *out = &D;
    return TGK_OK;
}

int routing_flags(tgk_routing* r, unsigned long long** out) {
    if (!r->flags) HCUDA(cudaMalloc(&r->flags, 4 * sizeof(unsigned long long)));
    *out = r->flags;
    return TGK_OK;
}

// Build (once per R) and upload the fused row-block plan of a scalar routing.
int ensure_plan(tgk_routing* rr, int R, const PlanDev** out, int C) {
    tgk_routing* r = rr->scalar ? rr->scalar : rr;
    if (C == 0) C = R;
    PlanDev* cache = nullptr;
    for (auto& pl : r->plan)
        if (pl.R == R && pl.C == C) {
            *out = &pl;
            return TGK_OK;
        }
    for (auto& pl : r->plan)
        if (pl.R == 0 && !cache) cache = &pl;
    if (!cache) {  // all slots in use: evict the first
        cache = &r->plan[0];
        cache->release();
    }
    PlanDev& D = *cache;
    const tgk_mesh* m = r->mesh;
    ScalarRoutingHost h;
    TGK_TRY(fetch_scalar_routing(r, h));
    auto& nodes = h.nodes;
    auto& conn = h.conn;
    auto& row_ptr = h.row_ptr;
    auto& vo = h.vo;
    auto& vs = h.vs;
    auto& slot = h.slot;
    PlanHost P;
    const int64_t lo = r->own_hi < 0 ? 0 : r->own_lo, hi = r->own_hi < 0 ? r->N : r->own_hi;
    const int64_t elo = r->elem_hi < 0 ? 0 : r->elem_lo, ehi = r->elem_hi < 0 ? r->E : r->elem_hi;
    TGK_TRY(build_plan(m->kind, m->N, m->E, nodes.data(), conn.data(), row_ptr.data(), vo.data(),
                       vs.data(), slot.data(), lo, hi, elo, ehi, R, C, P));
    D = PlanDev{};
    D.n_blocks = P.n_blocks;
    D.lmax = P.lmax;
    D.max_chunk_recs = P.max_chunk_recs;
    D.n_halo = static_cast<int64_t>(P.halo.size());
    D.n_records = static_cast<int64_t>(P.recs.size());
    for (int64_t b = 0; b < P.n_blocks; ++b) {
        D.max_block_halo = std::max<int>(D.max_block_halo, static_cast<int>(P.halo_off[b + 1] - P.halo_off[b]));
        D.max_block_chunks = std::max<int>(D.max_block_chunks, static_cast<int>(P.chunk_off[b + 1] - P.chunk_off[b]));
        D.max_block_recs = std::max<int>(
            D.max_block_recs, static_cast<int>(P.chunk_rec_off[P.chunk_off[b + 1]] - P.chunk_rec_off[P.chunk_off[b]]));
    }
    auto up = [&D](auto*& dst, const auto& v) -> int {
        using T = typename std::remove_reference<decltype(v)>::type::value_type;
        const size_t bytes = std::max<size_t>(16, v.size() * sizeof(T));
        HCUDA(cudaMalloc(reinterpret_cast<void**>(&dst), bytes));
        if (!v.empty()) HCUDA(cudaMemcpy(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
        D.bytes += static_cast<int64_t>(bytes);
        return TGK_OK;
    };
    TGK_TRY(up(D.row_off, P.row_off));
    TGK_TRY(up(D.rows, P.rows));
    TGK_TRY(up(D.rows_rp, P.rows_rp));
    TGK_TRY(up(D.halo_off, P.halo_off));
    TGK_TRY(up(D.halo, P.halo));
    TGK_TRY(up(D.bnode_off, P.bnode_off));
    TGK_TRY(up(D.bnodes, P.bnodes));
    TGK_TRY(up(D.halo_lconn, P.halo_lconn));
    D.max_bnodes = P.max_bnodes;
    TGK_TRY(up(D.chunk_off, P.chunk_off));
    TGK_TRY(up(D.chunk_rec_off, P.chunk_rec_off));
    TGK_TRY(up(D.chunk_row_off, P.chunk_row_off));
    TGK_TRY(up(D.recs, P.recs));
    D.R = R;
    D.C = C;
    *out = &D;
    return TGK_OK;
}

static int check_field(const tgk_field& f, const tgk_mesh* m, const char* what, int degree = 0) {
    if (f.type == TGK_FIELD_CONSTANT) return TGK_OK;
    if (f.type == TGK_FIELD_QUAD) {
        int Q = 0;
        TGK_TRY(tgk_tables(m->kind, degree, &Q, nullptr, nullptr, nullptr, nullptr));
        if (f.n != m->E * Q)
            return set_error(TGK_ERR_INPUT, std::string(what) + ": quadrature table: expected E x Q = " +
                                                std::to_string(m->E * Q) + " values, got " + std::to_string(f.n));
        return TGK_OK;
    }
    if (f.type == TGK_FIELD_ELEMENT) {
        if (f.n != m->E)
            return set_error(TGK_ERR_INPUT, std::string(what) + ": per-element coefficient: expected " +
                                                std::to_string(m->E) + " values, got " + std::to_string(f.n));
        return TGK_OK;
    }
    if (f.type == TGK_FIELD_NODAL) {
        if (f.n != m->N)
            return set_error(TGK_ERR_INPUT, std::string(what) + ": nodal field: expected " +
                                                std::to_string(m->N) + " values, got " + std::to_string(f.n));
        return TGK_OK;
    }
    return set_error(TGK_ERR_INPUT, std::string(what) + ": unknown field type");
}

// tg::assemble (physics.cpp:10-75) on device buffers
int assemble_dev(const tgk_problem* p, const tgk_mesh* m, tgk_routing* r, double* K, double* F,
                 double* M, cudaStream_t st, unsigned long long* d_bad) {
    if (!p || !m || !r) return set_error(TGK_ERR_INPUT, "tgk_assemble: null argument");
    if (p->mode != TGK_MODE_EXACT && p->mode != TGK_MODE_FAST)
        return set_error(TGK_ERR_INPUT, "tgk_assemble: unknown arithmetic mode");
    if (m->kind != TGK_TRI3 && m->kind != TGK_TET4)
        return set_error(TGK_ERR_INPUT, "P1 assembly supports TRI3 and TET4 meshes only");
    const int comps = p->kind == TGK_ELASTICITY ? m->d : 1;
    if (r->components != comps)
        return set_error(TGK_ERR_INPUT, "assemble: dofmap component count does not match problem kind");
    TGK_TRY(check_routing_fresh(m, r));
    // quadrature degree of physics.cpp:18-21 (the QUAD tables must be at it)
    const bool high = p->diffusion.type != TGK_FIELD_CONSTANT || p->kind == TGK_MASS || p->with_mass;
    const int degree = high ? 2 : 1;
    TGK_TRY(check_field(p->diffusion, m, "diffusion", degree));
    if (p->kind == TGK_ELASTICITY) {
        TGK_TRY(check_field(p->lambda, m, "lambda", degree));
        TGK_TRY(check_field(p->mu, m, "mu", degree));
        if (p->n_source > 0 && p->n_source != m->d)
            return set_error(TGK_ERR_INPUT, "elasticity body force needs one component per dimension");
    }
    for (int s = 0; s < std::min(p->n_source, 3); ++s) TGK_TRY(check_field(p->source[s], m, "source", degree));
    bool quad = p->diffusion.type == TGK_FIELD_QUAD;
    for (int s = 0; s < std::min(p->n_source, 3); ++s) quad = quad || p->source[s].type == TGK_FIELD_QUAD;
    if (p->kind == TGK_ELASTICITY) quad = quad || p->lambda.type == TGK_FIELD_QUAD || p->mu.type == TGK_FIELD_QUAD;
    if (p->with_mass && comps != 1)
        return set_error(TGK_ERR_INPUT, "mass matrix assembly only supported for scalar fields");
    TGK_TRY(host_ensure_device());
    if (p->kind == TGK_ELASTICITY) {
        // fused row-block kernel (fused_elast.cu); the materialised Stage I + II
        // path (evaluate -> local_stiffness_elasticity -> reduce_matrix) remains
        // behind TGK_ELAST_MATERIALISED=1 (needs a routing with segment maps)
        if (quad || getenv("TGK_ELAST_MATERIALISED")) return elasticity_assemble(p, m, r, K, F, st);
        if (p->mode == TGK_MODE_FAST) {
            const int rc = fast_elasticity_assemble(p, m, r, K, F, st);
            if (rc != kFastNotApplicable) return rc;
        }
        return fused_elasticity_assemble(p, m, r, K, F, st);
    }
    if (quad) return materialised_scalar_assemble(p, m, r, K, F, M, st, d_bad);
    if (p->mode == TGK_MODE_FAST) {
        const int rc = fast_scalar_assemble(p, m, r, K, F, M, st, d_bad);
        if (rc != kFastNotApplicable) return rc;
    }
    return fused_scalar_assemble(p, m, r, K, F, M, st, d_bad);
}

}  // namespace tgk

extern "C" {

int tgk_assemble_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, double* d_K,
                   double* d_F, double* d_M, void* stream) {
    return tgk::assemble_dev(p, m, const_cast<tgk_routing*>(r), d_K, d_F, d_M,
                             static_cast<cudaStream_t>(stream), nullptr);
}

// Batched assembly over coefficient fields (the north star's Map stage,
// batch.cpp:183-269 rerun per field as topopt.cpp:122-127 does): member b of
// the batch is `p` with every listed slot replaced by the per-element field
// data + b * stride.  Any problem kind and mode; outputs stacked member-major.
int tgk_assemble_fields_batched_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, int64_t B,
                                  const tgk_field_batch* fb, int n_fb, double* d_K, double* d_F, double* d_M,
                                  void* stream) {
    if (!p || !m || !r || (n_fb > 0 && !fb)) return set_error(TGK_ERR_INPUT, "assemble_fields_batched: null argument");
    if (B < 0 || n_fb < 0) return set_error(TGK_ERR_INPUT, "assemble_fields_batched: negative count");
    auto slot_field = [](tgk_problem& q, int slot) -> tgk_field* {
        switch (slot) {
            case TGK_SLOT_DIFFUSION: return &q.diffusion;
            case TGK_SLOT_LAMBDA: return &q.lambda;
            case TGK_SLOT_MU: return &q.mu;
            case TGK_SLOT_SOURCE0: case TGK_SLOT_SOURCE0 + 1: case TGK_SLOT_SOURCE0 + 2:
                return slot - TGK_SLOT_SOURCE0 < q.n_source ? &q.source[slot - TGK_SLOT_SOURCE0] : nullptr;
            default: return nullptr;
        }
    };
    tgk_problem q = *p;
    for (int i = 0; i < n_fb; ++i) {
        if (!slot_field(q, fb[i].slot))
            return set_error(TGK_ERR_INPUT, "assemble_fields_batched: field slot " + std::to_string(fb[i].slot) +
                                                " is not a field of this problem");
        if (!fb[i].data && B > 0) return set_error(TGK_ERR_INPUT, "assemble_fields_batched: null field data");
    }
    const int64_t nnz = r->nnz, N = r->N;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // scalar problems: one status word per member, read back once after the
    // batch (no host synchronisation per member); elasticity checks mu per call
    const bool async_status = p->kind != TGK_ELASTICITY && B > 0;
    unsigned long long* d_bads = nullptr;
    if (async_status) {
        TGK_TRY(host_ensure_device());
        HCUDA(cudaMalloc(&d_bads, sizeof(unsigned long long) * B));
    }
    std::unique_ptr<unsigned long long, cudaError_t (*)(void*)> guard(d_bads, cudaFree);
    if (async_status) HCUDA(cudaMemsetAsync(d_bads, 0xff, sizeof(unsigned long long) * B, st));
    for (int64_t b = 0; b < B; ++b) {
        for (int i = 0; i < n_fb; ++i) {
            const int64_t stride = fb[i].stride > 0 ? fb[i].stride : m->E;
            *slot_field(q, fb[i].slot) = tgk_field{TGK_FIELD_ELEMENT, 0.0, fb[i].data + b * stride, m->E};
        }
        TGK_TRY(tgk::assemble_dev(&q, m, const_cast<tgk_routing*>(r), d_K ? d_K + b * nnz : nullptr,
                                  d_F ? d_F + b * N : nullptr, d_M && q.with_mass ? d_M + b * nnz : nullptr, st,
                                  async_status ? d_bads + b : nullptr));
    }
    if (async_status) {
        std::vector<unsigned long long> h(static_cast<size_t>(B));
        HCUDA(cudaMemcpyAsync(h.data(), d_bads, sizeof(unsigned long long) * B, cudaMemcpyDeviceToHost, st));
        HCUDA(cudaStreamSynchronize(st));
        for (int64_t b = 0; b < B; ++b)  // the first failing member, as a per-field loop would report it
            if (h[static_cast<size_t>(b)] != ULLONG_MAX)
                return set_error(TGK_ERR_INPUT, "element " + std::to_string(h[static_cast<size_t>(b)]) +
                                                    " has non-positive Jacobian determinant");
    }
    return TGK_OK;
}

int tgk_assemble_f32_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, float* d_K, float* d_F,
                       float* d_M, unsigned long long* d_bad, void* stream) {
    if (!p || !m || !r) return set_error(TGK_ERR_INPUT, "tgk_assemble_f32_d: null argument");
    if (m->kind != TGK_TRI3 && m->kind != TGK_TET4)
        return set_error(TGK_ERR_INPUT, "P1 assembly supports TRI3 and TET4 meshes only");
    if (p->kind == TGK_ELASTICITY || r->components != 1)
        return set_error(TGK_ERR_INPUT, "tgk_assemble_f32_d: scalar problems only");
    TGK_TRY(tgk::check_routing_fresh(m, r));
    if (p->diffusion.type == TGK_FIELD_QUAD || (p->n_source > 0 && p->source[0].type == TGK_FIELD_QUAD))
        return set_error(TGK_ERR_INPUT, "tgk_assemble_f32_d: quadrature-table fields are fp64-only");
    TGK_TRY(check_field(p->diffusion, m, "diffusion"));
    for (int s = 0; s < std::min(p->n_source, 3); ++s) TGK_TRY(check_field(p->source[s], m, "source"));
    TGK_TRY(host_ensure_device());
    return tgk::fused_scalar_assemble_f32(p, m, const_cast<tgk_routing*>(r), d_K, d_F, d_M,
                                          static_cast<cudaStream_t>(stream), d_bad);
}

int tgk_allen_cahn_d(const tgk_mesh* m, const tgk_routing* r, const double* d_u, double eps, double* d_T,
                     double* d_F, void* stream) {
    if (!m || !r || !d_u || !d_T) return set_error(TGK_ERR_INPUT, "tgk_allen_cahn_d: null argument");
    if (m->kind != TGK_TRI3 && m->kind != TGK_TET4)
        return set_error(TGK_ERR_INPUT, "P1 assembly supports TRI3 and TET4 meshes only");
    if (r->components != 1) return set_error(TGK_ERR_INPUT, "AllenCahnStepper: scalar fields only");  // timestep.cpp:137
    TGK_TRY(tgk::check_routing_fresh(m, r));
    TGK_TRY(host_ensure_device());
    return tgk::fused_allen_cahn(m, const_cast<tgk_routing*>(r), d_u, eps, d_T, d_F, static_cast<cudaStream_t>(stream));
}

int tgk_assemble_async_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r,
                         double* d_K, double* d_F, double* d_M, unsigned long long* d_bad,
                         void* stream) {
    if (!d_bad) return set_error(TGK_ERR_INPUT, "tgk_assemble_async_d: d_bad is required");
    if (p && p->kind == TGK_ELASTICITY)
        return set_error(TGK_ERR_INPUT, "tgk_assemble_async_d: scalar problems only");
    return tgk::assemble_dev(p, m, const_cast<tgk_routing*>(r), d_K, d_F, d_M,
                             static_cast<cudaStream_t>(stream), d_bad);
}

// Host-buffer variant: field data and outputs on the host; copies inside.
int tgk_assemble(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, double* K,
                 double* F, double* M) {
    if (!p || !m || !r) return set_error(TGK_ERR_INPUT, "tgk_assemble: null argument");
    TGK_TRY(host_ensure_device());
    tgk_problem pd = *p;
    std::vector<void*> bufs;
    auto cleanup = [&bufs] {
        for (void* b : bufs) cudaFree(b);
    };
    auto upload = [&](tgk_field& f) -> int {
        if (f.type == TGK_FIELD_CONSTANT || !f.data) return TGK_OK;
        void* d = nullptr;
        HCUDA(cudaMalloc(&d, sizeof(double) * std::max<int64_t>(1, f.n)));
        bufs.push_back(d);
        HCUDA(cudaMemcpy(d, f.data, sizeof(double) * f.n, cudaMemcpyHostToDevice));
        f.data = static_cast<const double*>(d);
        return TGK_OK;
    };
    int rc = TGK_OK;
    rc = rc ? rc : upload(pd.diffusion);
    rc = rc ? rc : upload(pd.lambda);
    rc = rc ? rc : upload(pd.mu);
    for (int s = 0; s < std::min(pd.n_source, 3) && !rc; ++s) rc = upload(pd.source[s]);
    tgk_routing* rw = const_cast<tgk_routing*>(r);
    auto scratch = [&](double*& buf, int64_t n) -> int {
        if (buf) return TGK_OK;
        HCUDA(cudaMalloc(&buf, sizeof(double) * std::max<int64_t>(1, n)));
        return TGK_OK;
    };
    if (!rc) rc = scratch(rw->scratch_K, r->nnz);
    if (!rc) rc = scratch(rw->scratch_F, r->N);
    const bool want_m = p->with_mass && p->kind != TGK_MASS;  // a Mass problem returns no M (physics.cpp:25-31)
    if (!rc && want_m) rc = scratch(rw->scratch_M, r->nnz);
    double *dK = rw->scratch_K, *dF = rw->scratch_F, *dM = want_m ? rw->scratch_M : nullptr;
    if (!rc) rc = tgk::assemble_dev(&pd, m, rw, dK, dF, dM, nullptr, nullptr);
    if (!rc && K && cudaMemcpy(K, dK, sizeof(double) * r->nnz, cudaMemcpyDeviceToHost) != cudaSuccess) rc = set_error(TGK_ERR_CUDA, "copy K");
    if (!rc && F && cudaMemcpy(F, dF, sizeof(double) * r->N, cudaMemcpyDeviceToHost) != cudaSuccess) rc = set_error(TGK_ERR_CUDA, "copy F");
    if (!rc && M && dM && cudaMemcpy(M, dM, sizeof(double) * r->nnz, cudaMemcpyDeviceToHost) != cudaSuccess) rc = set_error(TGK_ERR_CUDA, "copy M");
    cleanup();
    return rc;
}

}  // extern "C"
