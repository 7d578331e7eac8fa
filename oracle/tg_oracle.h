/* TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 assembly path.
 *
 * A plain-C restatement of the reference's P1 Map/Reduce/adjoint algorithm
 * (arxiv 2602.05052 "TensorGalerkin", /root/reference/proj).  Each function
 * cites the reference file:line it restates and keeps the reference's
 * floating-point operation order (no FMA contraction: built with
 * -ffp-contract=off), so results are bit-identical to the reference library.
 * Pinned against the reference itself (oracle/_ref/libtgref.so) and the golden
 * fixtures in tests/golden/ by tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker.
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element kinds, same codes as tg::ElementKind (reference.hpp:10) */
enum { TGO_TRI3 = 0, TGO_QUAD4 = 1, TGO_TET4 = 2 };
/* local kernels (batch.hpp:41-87) */
enum {
    TGO_DIFFUSION = 0,   /* local_stiffness_diffusion, c1 = coeff E x Q          */
    TGO_ELASTICITY = 1,  /* local_stiffness_elasticity, c1 = lambda, c2 = mu     */
    TGO_MASS = 2,        /* local_mass, c1 = coeff                               */
    TGO_LOAD = 3,        /* local_load, c1 = source E x Q                        */
    TGO_LOAD_VECTOR = 4  /* local_load_vector, c1 = source E x Q x d             */
};
/* status codes: 0 ok, 1 numerical, 2 input (tg_main.cpp:979-988) */

typedef struct {
    int type; /* 0 constant, 1 per-element (E values), 2 nodal (N values) */
    double value;
    const double* data;
    int64_t n;
} tgo_field;

typedef struct tgo_routing tgo_routing;

const char* tgo_last_error(void);

int tgo_element_dim(int kind);
int tgo_element_nodes(int kind);
int tgo_default_degree(int kind, int mass);
/* reference_tables (reference.cpp:223-239); arrays may be NULL */
int tgo_tables(int kind, int degree, int* Q, double* points, double* weights, double* B,
               double* G);

/* generate_grid (mesh.cpp:96-169) without the boundary pass. */
void tgo_grid_sizes(int kind, const int64_t* div, int64_t* n_nodes, int64_t* n_elems);
int tgo_generate_grid(int kind, const double* ext, const int64_t* div, double* nodes,
                      int64_t* elems);
/* Mesh::content_hash (mesh.cpp:79-94) */
uint64_t tgo_content_hash(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                          int64_t n_elems);
/* build_dofmap (dofmap.cpp:9-25) */
void tgo_dofmap(int kind, const int64_t* elems, int64_t n_elems, int comps, int64_t* map);

/* batch_geometry + push_forward (batch.cpp:56-154).  Any output may be NULL.
 * Returns 2 and sets *bad to the smallest element with det <= 0. */
int tgo_geometry(int kind, const double* nodes, const int64_t* elems, int64_t n_elems,
                 int degree, double* jac, double* det, double* jac_invT, double* qpts,
                 double* grads, int64_t* bad);
/* The Stage-I local kernels (batch.cpp:156-312). */
int tgo_local(int kind, const double* nodes, const int64_t* elems, int64_t n_elems, int degree,
              int what, const double* c1, const double* c2, double* out, int64_t* bad);
/* CoefficientField::evaluate (coefficient.cpp:34-55) for constant/per-element/nodal */
int tgo_evaluate(int kind, const double* nodes, const int64_t* elems, int64_t n_elems,
                 int64_t n_nodes, int degree, const tgo_field* f, double* out);

/* build_routing (routing.cpp:12-85) over a DoF map (E x k). */
tgo_routing* tgo_routing_build(int64_t N, int64_t E, int k, const int64_t* map);
void tgo_routing_free(tgo_routing* r);
int64_t tgo_routing_nnz(const tgo_routing* r);
void tgo_routing_copy(const tgo_routing* r, int64_t* offsets, int64_t* cols, uint32_t* vec_off,
                      uint32_t* vec_slots, uint32_t* mat_off, uint32_t* mat_slots);
/* reduce_vector / reduce_matrix (routing.cpp:87-125) */
void tgo_reduce_vector(const tgo_routing* r, const double* local, double* F);
void tgo_reduce_matrix(const tgo_routing* r, const double* local, double* values);
/* scatter_add_oracle (routing.cpp:134-175) onto the routing's pattern */
void tgo_scatter_add(const tgo_routing* r, const int64_t* map, const double* localK,
                     const double* localF, double* values, double* F);

/* assemble (physics.cpp:10-75).  problem: 0 Poisson, 1 elasticity, 2 mass.
 * comps must match (1, or d for elasticity); routing built on that DoF map. */
int tgo_assemble(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                 int64_t n_elems, const tgo_routing* r, int problem, const tgo_field* diffusion,
                 const tgo_field* lambda, const tgo_field* mu, int plane_stress, int n_source,
                 const tgo_field* sources, int with_mass, double* K, double* F, double* M);

/* gradient_products (adjoint.cpp:68-82): dK[t] = lambda_i U_cols[t], dF = -lambda */
void tgo_gradient_products(const tgo_routing* r, const double* lambda, const double* U,
                           double* dK, double* dF);
/* Adjoint transpose gather, order of tg_main.cpp:846-850:
 * out[e] = sum_{a,b} (lambda[g_a] * K0[e,a,b]) * U[g_b] */
void tgo_adjoint_gather(int64_t E, int k, const int64_t* map, const double* K0,
                        const double* lambda, const double* U, double* out);
/* Pattern-generic chain rule of acceptance.cpp:372-377 (positive sign):
 * out[e] = sum_{a,b} dK[find(g_a,g_b)] * K0[e,a,b] */
void tgo_adjoint_generic(const tgo_routing* r, const int64_t* map, const double* K0,
                         const double* dK, double* out);

#ifdef __cplusplus
}
#endif
#endif
