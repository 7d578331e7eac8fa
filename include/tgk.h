/* tgk.h — C ABI of the B200-native P1 Galerkin assembly engine (libtgk.so).
 *
 * Drop-in boundary for the hot path of the reference library `tg`
 * (/root/reference/proj): Stage I "Map" (batch.hpp), Stage II "Reduce"
 * (routing.hpp), the whole-path entry tg::assemble (physics.hpp:55-56) and the
 * adjoint pieces (adjoint.hpp:27-28 + the per-element chain rule of
 * tests/acceptance.cpp:357-378 / tools/tg_main.cpp:840-856).  Each entry point
 * below cites the reference interface it replaces.  INTEGRATION.md shows the
 * binding a maintainer adds to bindings/module.cpp (pybind11) or a ctypes user.
 *
 * Conventions
 *  - plain C: opaque handles, pointers and sizes; no torch / CUDA types.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - "_d" suffix / d_ arguments: DEVICE pointers.  Functions without it take
 *    HOST pointers and do the host<->device copies themselves (synchronous,
 *    like the reference's std::vector API).
 *  - fp64 throughout; connectivity is int64 on the host side like tg::Mesh
 *    (mesh.hpp:19) and int32 on the device.
 *  - Status codes mirror the reference CLI (tools/tg_main.cpp:979-988):
 *    0 ok, 1 numerical (tg::NumericalError), 2 input (tg::InputError),
 *    3 CUDA / runtime failure.  tgk_last_error() gives the message; for a
 *    non-positive Jacobian it is "element <e> has non-positive Jacobian
 *    determinant" exactly like batch.cpp:124-126 (e = smallest such element).
 *  - No CPU fallback: every compute entry point fails with status 3 when no
 *    CUDA device is usable.
 */
#ifndef TGK_H
#define TGK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGK_OK 0
#define TGK_ERR_NUMERICAL 1
#define TGK_ERR_INPUT 2
#define TGK_ERR_CUDA 3

/* element kinds — same codes as tg::ElementKind (reference.hpp:10) */
#define TGK_TRI3 0
#define TGK_QUAD4 1 /* accepted by the host helpers only; P1 kernels are TRI3/TET4 */
#define TGK_TET4 2

/* problem kinds — tg::ProblemKind (physics.hpp:16) */
#define TGK_POISSON 0
#define TGK_ELASTICITY 1
#define TGK_MASS 2

/* coefficient field types — tg::CoefficientField variants (coefficient.hpp:17-50).
 * Analytic (a host std::function) has no device form: the caller evaluates it
 * (CoefficientField::evaluate, coefficient.cpp:34-55) and passes the quadrature
 * table (TGK_FIELD_QUAD). */
#define TGK_FIELD_CONSTANT 0
#define TGK_FIELD_ELEMENT 1 /* E values                       */
#define TGK_FIELD_NODAL 2   /* N_node values, interpolated by the basis (batch.cpp:314-333) */
#define TGK_FIELD_QUAD 3    /* E x Q values at the quadrature points of the degree assemble()
                               selects (physics.cpp:18-21): any CoefficientField, Analytic
                               included, evaluated by the caller; assembled through the
                               materialised Stage I + II kernels (bit-identical) */

/* arithmetic mode of tgk_problem (fp64 entries).
 *  TGK_MODE_EXACT: the reference operation order, no FMA contraction, CSR values
 *    bit-identical to the reference (ascending-element folds, row-block kernel).
 *  TGK_MODE_FAST: the north star's contract — pattern bit-exact, values within
 *    |dv| <= 1e-12 |v_ref| + 1e-14 max|v_ref|, bitwise
 *    deterministic run to run: FMA arithmetic, affine-P1 closed forms of the
 *    quadrature, a precomputed element-to-CSR-slot list per entry folded in a
 *    register (fast.cu).  Scalar problems with constant / per-element / nodal
 *    fields (a nodal mass coefficient, and elasticity, take the exact kernel).
 * The fp32 variant is a separate entry point (tgk_assemble_f32_d). */
#define TGK_MODE_EXACT 0
#define TGK_MODE_FAST 1

typedef struct tgk_mesh tgk_mesh;
typedef struct tgk_routing tgk_routing;

typedef struct {
    int type;           /* TGK_FIELD_* */
    double value;       /* TGK_FIELD_CONSTANT */
    const double* data; /* TGK_FIELD_ELEMENT / TGK_FIELD_NODAL (host or device per entry point) */
    int64_t n;          /* number of values in data */
} tgk_field;

/* ProblemSpec (physics.hpp:20-45), assembly-relevant members only. */
typedef struct {
    int kind;              /* TGK_POISSON / TGK_ELASTICITY / TGK_MASS */
    tgk_field diffusion;   /* Poisson / mass coefficient */
    tgk_field lambda, mu;  /* elasticity Lame fields */
    int plane_stress;      /* 2D elasticity only */
    int n_source;          /* 0, 1 (scalar) or d (elasticity body force) */
    tgk_field source[3];
    int with_mass;         /* also assemble M (scalar problems only; physics.cpp:68-73) */
    int mode;              /* TGK_MODE_EXACT or TGK_MODE_FAST (other values: status 2) */
} tgk_problem;

/* Routing description (RoutingMatrices, routing.hpp:16-32).  All pointers are
 * DEVICE pointers owned by the routing handle.  Segment maps are present only
 * when the routing was built with TGK_ROUTING_SEGMENTS. */
typedef struct {
    int64_t N, E, nnz;
    int k, components;
    const int64_t* row_ptr;      /* CsrPattern::offsets, N+1 */
    const int64_t* col_idx;      /* CsrPattern::cols, nnz */
    const uint32_t* slot_of;     /* element-to-CSR-slot map, E*k*k: slot_of[(e*k+a)*k+b] = t
                                    (inverse of mat_slots); components==1 only */
    const uint32_t* vec_offsets; /* N+1 */
    const uint32_t* vec_slots;   /* E*k   */
    const uint32_t* mat_offsets; /* nnz+1 */
    const uint32_t* mat_slots;   /* E*k*k */
} tgk_routing_view;

#define TGK_ROUTING_SEGMENTS 1 /* also build vec_/mat_ segment maps (reference layout) */

/* ------------------------------------------------------------------ misc */
const char* tgk_last_error(void);
int tgk_version(void);
int tgk_device_count(void);  /* 0 on a host without a usable GPU */
/* tg::set_thread_count (parallel.hpp:9) — accepted for API parity; the GPU
 * path's results never depend on it (parallel.hpp:12-14). */
void tgk_set_thread_count(int n);
int tgk_thread_count(void);

/* ------------------------------------------------------------------ host helpers (CPU) */
/* tg::generate_grid (mesh.cpp:96-169) — bit-identical node/element arrays.
 * Query sizes with nodes == elems == NULL. */
int tgk_grid_sizes(int kind, const int64_t* divisions, int64_t* n_nodes, int64_t* n_elems);
int tgk_generate_grid(int kind, const double* extents, const int64_t* divisions, double* nodes,
                      int64_t* elems);
/* Mesh::content_hash (mesh.cpp:79-94) */
uint64_t tgk_content_hash(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                          int64_t n_elems);
/* topological_boundary (mesh.cpp:185-209): sorted boundary node ids; returns count,
 * writes when out != NULL. */
int64_t tgk_topological_boundary(int kind, const int64_t* elems, int64_t n_elems,
                                 int64_t n_nodes, int64_t* out);
/* Mesh::validate (mesh.cpp:56-77) */
int tgk_validate(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                 int64_t n_elems);
/* quadrature tables (reference.cpp:223-247) */
int tgk_default_degree(int kind, int mass);
int tgk_tables(int kind, int degree, int* Q, double* points, double* weights, double* B,
               double* G);

/* ------------------------------------------------------------------ mesh */
/* Upload a tg::Mesh (host arrays, int64 connectivity) to the device. */
int tgk_mesh_create(int kind, const double* nodes, int64_t n_nodes, const int64_t* elems,
                    int64_t n_elems, tgk_mesh** out);
/* Wrap device arrays (node-major fp64 coordinates, int32 connectivity); not owned.
 * The caller must not change the connectivity of a wrapped mesh that has
 * routings, and must call tgk_mesh_coordinates_changed() after changing its
 * coordinates in place (the fused kernels certify coordinates once). */
int tgk_mesh_create_d(int kind, const double* d_nodes, int64_t n_nodes, const int32_t* d_elems,
                      int64_t n_elems, tgk_mesh** out);
/* Re-upload host arrays (either may be NULL) into an existing mesh of the same
 * sizes (timed e2e path).  New coordinates are re-certified on the next call;
 * connectivity that DIFFERS from the current one marks every routing built
 * from this mesh stale: they then fail with status 2 until rebuilt. */
int tgk_mesh_upload(tgk_mesh* m, const double* nodes, const int64_t* elems, void* stream);
/* Stream-ordered tgk_mesh_upload for pipelined host-to-host loops: no host
 * synchronisation inside.  The connectivity's range check (mesh.cpp:61-64) and
 * change detection run on the device and accumulate until
 * tgk_mesh_upload_check(), which waits for the device, reports an out-of-range
 * node id (status 2) and marks the mesh's routings stale if the connectivity
 * changed.  Until then, out-of-range ids are stored as node 0 (memory-safe)
 * and assemblies on a mesh whose connectivity changed use the routings and
 * plans of the previous connectivity. */
int tgk_mesh_upload_async(tgk_mesh* m, const double* nodes, const int64_t* elems, void* stream);
int tgk_mesh_upload_check(tgk_mesh* m);
/* Coordinates of a wrapped (tgk_mesh_create_d) mesh were changed in place. */
int tgk_mesh_coordinates_changed(tgk_mesh* m);
void tgk_mesh_destroy(tgk_mesh* m);
int tgk_mesh_info(const tgk_mesh* m, int* kind, int64_t* n_nodes, int64_t* n_elems,
                  const double** d_nodes, const int32_t** d_elems);

/* ------------------------------------------------------------------ routing */
/* build_dofmap (dofmap.cpp:9-25) + build_routing (routing.cpp:12-85) on the GPU.
 * CSR pattern and slot map are bit-identical to the reference.  components is
 * 1 or the mesh dimension.  flags: TGK_ROUTING_SEGMENTS. */
int tgk_routing_build(const tgk_mesh* m, int components, int flags, void* stream,
                      tgk_routing** out);
void tgk_routing_destroy(tgk_routing* r);
int tgk_routing_get_view(const tgk_routing* r, tgk_routing_view* out);
/* Copy the reference-layout arrays to host (any pointer may be NULL). */
int tgk_routing_copy(const tgk_routing* r, int64_t* row_ptr, int64_t* col_idx, uint32_t* slot_of,
                     uint32_t* vec_offsets, uint32_t* vec_slots, uint32_t* mat_offsets,
                     uint32_t* mat_slots);
/* Device routing from a caller's RoutingMatrices host arrays (routing.hpp:16-32:
 * pattern offsets / cols, vec_ and mat_ segment maps) — the drop-in keeps the
 * caller's routing instead of rebuilding it.  Sizes must match the mesh
 * (N = N_node * components, k = k_geom * components). */
int tgk_routing_create_host(const tgk_mesh* m, int components, int64_t N, int64_t E, int k, int64_t nnz,
                            const int64_t* row_ptr, const int64_t* col_idx, const uint32_t* vec_offsets,
                            const uint32_t* vec_slots, const uint32_t* mat_offsets, const uint32_t* mat_slots,
                            void* stream, tgk_routing** out);
/* Row-owning partitions: restrict the fused assembly to the scalar (node)
 * rows [row_lo, row_hi) of this routing; elements incident to them are
 * recomputed as halo.  Other output rows are left untouched.  Resets the plan. */
int tgk_routing_set_owned_rows(tgk_routing* r, int64_t row_lo, int64_t row_hi);
/* Multi-GPU slabs with an interface exchange: restrict the fused assembly to
 * the elements [elem_lo, elem_hi).  Rows touched only by other elements come
 * out as +0.0; rows shared with other elements hold the partial left fold of
 * these elements (to be summed with the other ranks' partials).  Resets the plan. */
int tgk_routing_set_element_range(tgk_routing* r, int64_t elem_lo, int64_t elem_hi);
/* Interface sum of the multi-GPU exchange (paper_2602_05052_b200/dist.py):
 * d_values[i] = d_lower[i] + d_values[i] for i < n (device pointers). */
int tgk_interface_combine_d(const double* d_lower, double* d_values, int64_t n, void* stream);
/* Fused-plan statistics for blocks of rows_per_block (128 or 256) rows (builds
 * the plan if needed): CUDA blocks, halo elements (halo / E = recompute
 * factor), packed records, device bytes. */
int tgk_routing_plan_stats(tgk_routing* r, int rows_per_block, int64_t* n_blocks, int64_t* n_halo,
                           int64_t* n_records, int64_t* bytes);
/* Fast-mode plan of the latest TGK_MODE_FAST assembly on this routing
 * (plan_fast.cpp): rows per block, blocks, halo elements (halo / E = recompute
 * factor), CSR entries folded (after the symmetric dedup, padded), item words,
 * device bytes.  Status 2 before the first fast-mode assembly. */
int tgk_routing_fast_plan_info(const tgk_routing* r, int* rows_per_block, int64_t* n_blocks, int64_t* n_halo,
                               int64_t* n_entries, int64_t* n_words, int64_t* bytes);
/* Routing cache file in the reference layout ("tg-rout2", save_routing routing.cpp:194-209). */
int tgk_routing_save(const tgk_routing* r, uint64_t mesh_hash, const char* path);
/* load_routing (routing.cpp:211-234): *hit = 0 (status 0) on a missing file or a
 * magic / mesh-hash / size mismatch, as the reference returns false; else a
 * device routing bit-identical to the cached arrays in *out. */
int tgk_routing_load(const tgk_mesh* m, int components, uint64_t mesh_hash, const char* path, void* stream,
                     int* hit, tgk_routing** out);

/* ------------------------------------------------------------------ Stage I (Map), materialised */
/* batch_geometry + push_forward (batch.cpp:56-154).  Outputs E x Q x ... like
 * GeometryBatch/PhysicalGradients; any may be NULL.  Device pointers. */
int tgk_geometry_d(const tgk_mesh* m, int degree, double* d_jac, double* d_det,
                   double* d_jac_invT, double* d_qpts, double* d_grads, void* stream);
/* local_stiffness_diffusion (batch.cpp:156-181): coeff E x Q table, out E x k x k */
int tgk_local_stiffness_diffusion_d(const tgk_mesh* m, int degree, const double* d_coeff_eq,
                                    double* d_out, void* stream);
/* local_stiffness_elasticity (batch.cpp:183-248): out E x (k d) x (k d) */
int tgk_local_stiffness_elasticity_d(const tgk_mesh* m, int degree, const double* d_lambda_eq,
                                     const double* d_mu_eq, double* d_out, void* stream);
/* local_mass (batch.cpp:250-269) */
int tgk_local_mass_d(const tgk_mesh* m, int degree, const double* d_coeff_eq, double* d_out,
                     void* stream);
/* local_load (batch.cpp:271-289) */
int tgk_local_load_d(const tgk_mesh* m, int degree, const double* d_source_eq, double* d_out,
                     void* stream);
/* local_load_vector (batch.cpp:291-312): source E x Q x d */
int tgk_local_load_vector_d(const tgk_mesh* m, int degree, const double* d_source_eqc,
                            double* d_out, void* stream);
/* CoefficientField::evaluate (coefficient.cpp:34-55) for constant / element / nodal
 * fields (field data on the device): out E x Q */
int tgk_evaluate_field_d(const tgk_mesh* m, int degree, const tgk_field* f, double* d_out,
                         void* stream);

/* ------------------------------------------------------------------ Stage II (Reduce), materialised */
/* reduce_matrix / reduce_vector (routing.cpp:87-125): needs TGK_ROUTING_SEGMENTS.
 * Bitwise identical to the reference (ascending-slot left fold per output). */
int tgk_reduce_matrix_d(const tgk_routing* r, const double* d_local, double* d_values,
                        void* stream);
int tgk_reduce_vector_d(const tgk_routing* r, const double* d_local, double* d_F, void* stream);

/* scatter_add_oracle (routing.cpp:134-175): the reference's independent
 * correctness baseline — its own pattern and a per-element scatter in element
 * order — by a different GPU algorithm than tgk_routing_build (one stable
 * radix sort of all (row, col) contribution keys).  HOST buffers: call with
 * offsets = cols = values = NULL to get *nnz, then with N+1 / nnz / nnz
 * arrays; local_vectors (E x k) and F (N) may be NULL.  Bit-identical. */
int tgk_scatter_add(const tgk_mesh* m, const double* local_matrices, const double* local_vectors, int64_t* nnz,
                    int64_t* offsets, int64_t* cols, double* values, double* F);

/* ------------------------------------------------------------------ fused assembly */
/* tg::assemble (physics.cpp:10-75): Map fused with Reduce — local tensors
 * never touch HBM.  Writes K values (nnz), F (N) and, with with_mass, M values.
 * Field data pointers in *p are DEVICE pointers.  Output pattern is the
 * routing's (K, M and dK share one CsrPattern, adjoint.cpp:73). */
int tgk_assemble_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r,
                   double* d_K, double* d_F, double* d_M, void* stream);
/* Asynchronous variant for streams / CUDA-graph capture (scalar problems):
 * no host synchronisation; the smallest element with det <= 0 (or ~0ull when
 * none) is written to the 8-byte DEVICE word *d_bad for the caller to check. */
int tgk_assemble_async_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r,
                         double* d_K, double* d_F, double* d_M, unsigned long long* d_bad,
                         void* stream);
/* fp32 variant of tgk_assemble_d for scalar problems: the same fused kernel in
 * single precision with float CSR values / load (field data stays fp64 and is
 * rounded on load).  Accuracy vs the fp64 reference: |dv| <= 1e-5 |v| + 1e-7 max|v|
 * (north star "1e-5 in fp32"). */
int tgk_assemble_f32_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, float* d_K,
                       float* d_F, float* d_M, unsigned long long* d_bad, void* stream);
/* d_bad: NULL = check the Jacobians synchronously; else asynchronous, the smallest
 * element with det <= 0 (or ~0ull) lands in the 8-byte device word *d_bad. */
/* Same call on HOST buffers (field data, outputs), with the copies inside. */
int tgk_assemble(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, double* K,
                 double* F, double* M);

/* Batched operator-learning assembly: B per-element coefficient fields
 * (d_rho, B x E, field-major) on one mesh -> B stiffness value arrays
 * (d_K, B x nnz) and, if d_F != NULL, one load vector for the constant source
 * `source`.  Same arithmetic as assemble() with diffusion = per_element(rho_b). */
int tgk_assemble_batched_d(const tgk_mesh* m, const tgk_routing* r, int64_t B,
                           const double* d_rho, double source, double* d_K, double* d_F,
                           int mode, void* stream);

/* Batched assembly over coefficient fields, any problem kind (Poisson, mass,
 * elasticity) and mode: batch member b is *p with each listed slot replaced by
 * the per-element field (device) fb[i].data + b * fb[i].stride (stride 0: E).
 * Outputs are stacked member-major: d_K B x nnz, d_F B x N (may be NULL),
 * d_M B x nnz (p->with_mass; may be NULL).  Each member's arithmetic is that
 * of tgk_assemble_d on the same problem (exact: bit-identical to tg::assemble). */
#define TGK_SLOT_DIFFUSION 0
#define TGK_SLOT_LAMBDA 1
#define TGK_SLOT_MU 2
#define TGK_SLOT_SOURCE0 3 /* +c: body-force component c (c < n_source) */
typedef struct {
    int slot;           /* TGK_SLOT_* */
    const double* data; /* device, per-element values of member 0 */
    int64_t stride;     /* values between consecutive members (0: E) */
} tgk_field_batch;
int tgk_assemble_fields_batched_d(const tgk_problem* p, const tgk_mesh* m, const tgk_routing* r, int64_t B,
                                  const tgk_field_batch* fb, int n_fb, double* d_K, double* d_F, double* d_M,
                                  void* stream);

/* Allen-Cahn Newton re-assembly (AllenCahnStepper::step, timestep.cpp:144-178;
 * SURVEY.md 8(f) rank 1), fused in one pass at the mass degree for the nodal
 * state u (N values, device):
 *   d_T = reduce_matrix(local_mass(reaction_tangent_coefficient(u, eps)))  (nnz)
 *   d_F = reduce_vector(local_reaction_load(u, eps))                       (N; may be NULL)
 * (batch.cpp:314-351).  Bit-identical to the reference. */
int tgk_allen_cahn_d(const tgk_mesh* m, const tgk_routing* r, const double* d_u, double eps, double* d_T,
                     double* d_F, void* stream);

/* ------------------------------------------------------------------ adjoint */
/* gradient_products (adjoint.cpp:68-82): dK[t] = lambda_i U_cols[t] on the
 * pattern, dF = -lambda.  Batched over B fields (lambda, U: B x N). */
int tgk_gradient_products_d(const tgk_routing* r, int64_t B, const double* d_lambda,
                            const double* d_U, double* d_dK, double* d_dF, void* stream);
/* Fused adjoint transpose gather (chain rule of tg_main.cpp:846-850 and
 * acceptance.cpp:372-377): for each field b and element e,
 *   out[b,e] = sum_{a,c} (lambda_b[g_a] * K0_e[a,c]) * U_b[g_c]
 * with K0_e the unit-coefficient local diffusion stiffness at the stiffness
 * degree, recomputed in registers (dK and K0 are never materialised).
 * lambda, U: B x N (N = routing.N); out: B x E. */
int tgk_adjoint_gather_d(const tgk_mesh* m, const tgk_routing* r, int64_t B,
                         const double* d_lambda, const double* d_U, double* d_out, int degree,
                         void* stream);

/* simp_sensitivity (adjoint.cpp:101-125): for every element
 * sens[e] = -p rho_e^(p-1) (E_max - E_min) u_e^T K0_e u_e, u_e[a] = U[map[e k + a]],
 * in the reference's operation order (bit-identical for p = 3; pow otherwise).
 * Any element kind / component count: d_map is the DofMap's E x k element-to-DoF
 * array (device int64), d_unit_stiffness the E x k x k unit-coefficient local
 * stiffness (device), d_U the n_dofs solution.  k in [1, 32]; a DoF index outside
 * [0, n_dofs) -> status 2. */
int tgk_simp_sensitivity_d(int64_t E, int k, const int64_t* d_map, const double* d_rho, double p, double E_min,
                           double E_max, const double* d_unit_stiffness, const double* d_U, int64_t n_dofs,
                           double* d_sens, void* stream);

/* ------------------------------------------------------------------ consumers of the CSR */
typedef struct tgk_condensed tgk_condensed;
/* SparseOperator::apply (sparse.cpp:18-31): y = A x, row sums in column order from +0.0. */
int tgk_spmv_d(int64_t rows, const int64_t* d_offsets, const int64_t* d_cols, const double* d_values,
               const double* d_x, double* d_y, void* stream);
/* condense (solver.cpp:34-85) on device CSR (N rows, CsrPattern offsets/cols, K values, F):
 * free / constrained DoF lists (ascending), K_ff pattern and values, F_f = F - K_fc g.
 * Duplicate Dirichlet DoFs: the last value wins (as the reference's assignment loop).
 * Out-of-range DoF -> status 2 "condense: dirichlet dof out of range". */
int tgk_condense_d(int64_t N, const int64_t* d_offsets, const int64_t* d_cols, const double* d_K, const double* d_F,
                   int64_t n_dirichlet, const int64_t* d_dofs, const double* d_values, void* stream,
                   tgk_condensed** out);
int tgk_condensed_info(const tgk_condensed* c, int64_t* n_free, int64_t* n_fixed, int64_t* nnz_ff,
                       const int64_t** d_free_dofs, const int64_t** d_fixed_dofs, const double** d_prescribed,
                       const int64_t** d_offsets, const int64_t** d_cols, const double** d_values,
                       const double** d_F_f);
/* Copy the condensed system to host arrays (any pointer may be NULL). */
int tgk_condensed_copy(const tgk_condensed* c, int64_t* free_dofs, int64_t* fixed_dofs, double* prescribed,
                       int64_t* offsets, int64_t* cols, double* values, double* F_f);
/* restrict_to_free (solver.cpp:87-103): the free-free block of another operator on the same pattern. */
int tgk_restrict_to_free_d(const tgk_condensed* c, const int64_t* d_offsets, const int64_t* d_cols, const double* d_A,
                           double* d_out, void* stream);
/* CondensedSystem::expand (solver.cpp:20-26): full vector from free values + prescribed values. */
int tgk_expand_d(const tgk_condensed* c, const double* d_u_free, double* d_u, void* stream);
void tgk_condensed_destroy(tgk_condensed* c);
/* Device-to-device copy on a stream (plumbing for the Python layer). */
int tgk_copy_d2d(void* dst, const void* src, int64_t nbytes, void* stream);
/* Device memory plumbing for host-language callers without the CUDA runtime
 * headers (adapter/physics_gpu.cpp, ctypes): cudaMalloc / cudaFree / blocking copies. */
int tgk_alloc_d(void** p, int64_t nbytes);
int tgk_free_d(void* p);
int tgk_copy_d2h(void* dst, const void* src, int64_t nbytes);
int tgk_copy_h2d(void* dst, const void* src, int64_t nbytes);
/* bicgstab (solver.cpp:105-227): Jacobi-preconditioned BiCGSTAB with up to 8
 * restarts, divergence rollback and best-iterate fallback, on device CSR.
 * d_x holds the initial guess and receives the solution.  Dot products are
 * deterministic fixed-order reductions (the reference folds serially), so
 * iterates agree with the reference to rounding, not bitwise.
 * Zero diagonal -> status 1 (NumericalError) like the reference. */
int tgk_bicgstab_d(int64_t n, const int64_t* d_offsets, const int64_t* d_cols, const double* d_values,
                   const double* d_b, double* d_x, double tol_rel, double tol_abs, int64_t max_iter,
                   int64_t* iterations, double* rel_residual, int* converged, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TGK_H */
