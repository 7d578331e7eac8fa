// `_tgfem`: the reference's compiled Python module (proj/bindings/module.cpp:54-196,
// imported by proj/python/tgfem/__init__.py and proj/tests/test_python_smoke.py)
// rebuilt over libtgk's C ABI (include/tgk.h): same module name, functions,
// argument names and defaults, return types and exception classes, with the
// assembly path computed by the sm_100a kernels.  A caller that puts this
// module's directory first on sys.path gets the GPU path without code changes.
//
// Differences by design (as in paper_2602_05052_b200/tgfem.py):
//  - the device mesh and the routing are built once per Mesh object and reused
//    (the reference rebuilds build_dofmap / build_routing on every call,
//    module.cpp:116-117, 124-125, 141-142);
//  - solve_poisson uses the device BiCGSTAB at every size (no dense-LU branch);
//  - load_gmsh / write_gmsh delegate to the MSH 4.1 reader / writer of
//    paper_2602_05052_b200.tgfem; topopt_cantilever (SIMP on QUAD4) is outside
//    the accelerated path and raises NotImplementedError.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgk.h"

namespace py = pybind11;

namespace {

struct InputError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// tgk status -> the reference's exception classes (errors.hpp)
void check(int rc) {
    if (rc == TGK_OK) return;
    const std::string msg = tgk_last_error();
    if (rc == TGK_ERR_INPUT) throw InputError(msg);
    if (rc == TGK_ERR_NUMERICAL) throw NumericalError(msg);
    throw std::runtime_error("libtgk: " + msg);
}

int kind_code(const std::string& name) {
    if (name == "tri3") return TGK_TRI3;
    if (name == "quad4") return TGK_QUAD4;
    if (name == "tet4") return TGK_TET4;
    throw InputError("unknown element kind: " + name);
}
const char* kind_name(int kind) { return kind == TGK_TRI3 ? "tri3" : kind == TGK_QUAD4 ? "quad4" : "tet4"; }
int nodes_per_element(int kind) { return kind == TGK_TRI3 ? 3 : 4; }

// Device buffer (tgk_alloc_d / tgk_free_d: no CUDA runtime headers here).
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { check(tgk_alloc_d(&p, static_cast<int64_t>(bytes ? bytes : 8))); }
    DevBuf(const void* host, size_t bytes) : DevBuf(bytes) {
        if (bytes) check(tgk_copy_h2d(p, host, static_cast<int64_t>(bytes)));
    }
    ~DevBuf() {
        if (p) tgk_free_d(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    template <class T>
    void to_host(T* dst, size_t n) const {
        if (n) check(tgk_copy_d2h(dst, p, static_cast<int64_t>(n * sizeof(T))));
    }
};

// tg::Mesh (mesh.hpp:15-41) plus its lazily built device state.
class Mesh {
public:
    Mesh(int kind, std::vector<double> nodes, std::vector<int64_t> elems, std::vector<int64_t> boundary)
        : kind_(kind), nodes_(std::move(nodes)), elems_(std::move(elems)), boundary_(std::move(boundary)) {}
    ~Mesh() {
        if (routing_) tgk_routing_destroy(routing_);
        if (dev_) tgk_mesh_destroy(dev_);
    }
    Mesh(const Mesh&) = delete;
    Mesh& operator=(const Mesh&) = delete;

    int kind() const { return kind_; }
    int dim() const { return kind_ == TGK_TET4 ? 3 : 2; }
    int k() const { return nodes_per_element(kind_); }
    int64_t node_count() const { return static_cast<int64_t>(nodes_.size()) / dim(); }
    int64_t element_count() const { return static_cast<int64_t>(elems_.size()) / k(); }
    const std::vector<double>& nodes() const { return nodes_; }
    const std::vector<int64_t>& elements() const { return elems_; }
    const std::vector<int64_t>& boundary_nodes() {
        if (boundary_.empty() && !elems_.empty()) {  // topological_boundary (mesh.cpp:185-209)
            const int64_t n = tgk_topological_boundary(kind_, elems_.data(), element_count(), node_count(), nullptr);
            if (n < 0) check(TGK_ERR_INPUT);
            boundary_.resize(static_cast<size_t>(n));
            tgk_topological_boundary(kind_, elems_.data(), element_count(), node_count(), boundary_.data());
        }
        return boundary_;
    }
    uint64_t content_hash() const {
        return tgk_content_hash(kind_, nodes_.data(), node_count(), elems_.data(), element_count());
    }
    tgk_mesh* device() {
        if (kind_ != TGK_TRI3 && kind_ != TGK_TET4)
            throw InputError("P1 assembly supports TRI3 and TET4 meshes only");
        if (!dev_) check(tgk_mesh_create(kind_, nodes_.data(), node_count(), elems_.data(), element_count(), &dev_));
        return dev_;
    }
    // scalar DoF map + routing with the reference's segment maps
    tgk_routing* routing() {
        if (!routing_) check(tgk_routing_build(device(), 1, TGK_ROUTING_SEGMENTS, nullptr, &routing_));
        return routing_;
    }

private:
    int kind_;
    std::vector<double> nodes_;
    std::vector<int64_t> elems_;
    std::vector<int64_t> boundary_;
    tgk_mesh* dev_ = nullptr;
    tgk_routing* routing_ = nullptr;
};

template <class T>
py::array_t<T> to_array(const std::vector<T>& v) {
    return py::array_t<T>(static_cast<py::ssize_t>(v.size()), v.data());
}

std::vector<double> from_array(const py::array_t<double, py::array::c_style | py::array::forcecast>& a) {
    return std::vector<double>(a.data(), a.data() + a.size());
}

std::shared_ptr<Mesh> make_grid(const std::string& kind, const std::vector<double>& extents,
                                const std::vector<int64_t>& divisions) {
    const int code = kind_code(kind);
    const size_t d = code == TGK_TET4 ? 3 : 2;
    if (extents.size() != d || divisions.size() != d)
        throw InputError("generate_grid: extents/divisions must have " + std::to_string(d) + " entries for " + kind);
    int64_t nn = 0, ne = 0;
    check(tgk_grid_sizes(code, divisions.data(), &nn, &ne));
    std::vector<double> nodes(static_cast<size_t>(nn) * d);
    std::vector<int64_t> elems(static_cast<size_t>(ne) * nodes_per_element(code));
    check(tgk_generate_grid(code, extents.data(), divisions.data(), nodes.data(), elems.data()));
    return std::make_shared<Mesh>(code, std::move(nodes), std::move(elems), std::vector<int64_t>{});
}

// reduce_matrix / scatter_add_oracle result: SparseOperator as a dict (module.cpp csr_dict)
py::dict csr_dict(int64_t rows, const std::vector<int64_t>& offsets, const std::vector<int64_t>& cols,
                  const std::vector<double>& values) {
    py::dict d;
    d["rows"] = rows;
    d["offsets"] = to_array(offsets);
    d["cols"] = to_array(cols);
    d["values"] = to_array(values);
    return d;
}

py::dict routing_csr(tgk_routing* r, const std::vector<double>& values) {
    tgk_routing_view v{};
    check(tgk_routing_get_view(r, &v));
    std::vector<int64_t> off(static_cast<size_t>(v.N) + 1), cols(static_cast<size_t>(v.nnz));
    check(tgk_routing_copy(r, off.data(), cols.data(), nullptr, nullptr, nullptr, nullptr, nullptr));
    return csr_dict(v.N, off, cols, values);
}

// batched diffusion stiffness blocks, E x k x k (module.cpp:92-112; batch.cpp:156-181)
py::array_t<double> local_stiffness(Mesh& mesh, py::object coeff) {
    tgk_mesh* m = mesh.device();
    const int degree = tgk_default_degree(mesh.kind(), 0);
    int Q = 0;
    check(tgk_tables(mesh.kind(), degree, &Q, nullptr, nullptr, nullptr, nullptr));
    const int64_t E = mesh.element_count();
    const int k = mesh.k();
    std::vector<double> c(static_cast<size_t>(E) * Q, 1.0);
    if (!coeff.is_none()) {  // CoefficientField::per_element (coefficient.cpp:34-55)
        const auto pe = from_array(coeff.cast<py::array_t<double, py::array::c_style | py::array::forcecast>>());
        if (static_cast<int64_t>(pe.size()) != E)
            throw InputError("per-element coefficient: expected " + std::to_string(E) + " values, got " +
                             std::to_string(pe.size()));
        for (int64_t e = 0; e < E; ++e)
            for (int q = 0; q < Q; ++q) c[static_cast<size_t>(e) * Q + q] = pe[static_cast<size_t>(e)];
    }
    DevBuf dc(c.data(), c.size() * sizeof(double)), dout(static_cast<size_t>(E) * k * k * sizeof(double));
    check(tgk_local_stiffness_diffusion_d(m, degree, dc.as<double>(), dout.as<double>(), nullptr));
    py::array_t<double> out({static_cast<py::ssize_t>(E), static_cast<py::ssize_t>(k), static_cast<py::ssize_t>(k)});
    dout.to_host(out.mutable_data(), static_cast<size_t>(E) * k * k);
    return out;
}

// reduce_matrix (routing.cpp:109-124) on the routing's segment maps
py::dict reduce_matrix(Mesh& mesh, const py::array_t<double, py::array::c_style | py::array::forcecast>& local) {
    tgk_routing* r = mesh.routing();
    tgk_routing_view v{};
    check(tgk_routing_get_view(r, &v));
    if (local.size() != v.E * v.k * v.k) throw InputError("reduce_matrix: local tensor shape mismatch");
    DevBuf dl(local.data(), static_cast<size_t>(local.size()) * sizeof(double));
    DevBuf dv(static_cast<size_t>(v.nnz) * sizeof(double));
    check(tgk_reduce_matrix_d(r, dl.as<double>(), dv.as<double>(), nullptr));
    std::vector<double> values(static_cast<size_t>(v.nnz));
    dv.to_host(values.data(), values.size());
    return routing_csr(r, values);
}

// scatter_add_oracle (routing.cpp:134-175): its own pattern and per-element
// scatter, by an algorithm independent of the routing build (tgk_scatter_add)
py::dict scatter_add_oracle(Mesh& mesh, const py::array_t<double, py::array::c_style | py::array::forcecast>& local) {
    const int k = mesh.k();
    if (local.size() != mesh.element_count() * k * k)
        throw InputError("scatter_add_oracle: local tensor shape mismatch");
    tgk_mesh* m = mesh.device();
    int64_t nnz = 0;
    check(tgk_scatter_add(m, local.data(), nullptr, &nnz, nullptr, nullptr, nullptr, nullptr));
    const int64_t n = mesh.node_count();
    std::vector<int64_t> off(static_cast<size_t>(n) + 1), cols(static_cast<size_t>(nnz));
    std::vector<double> values(static_cast<size_t>(nnz));
    check(tgk_scatter_add(m, local.data(), nullptr, &nnz, off.data(), cols.data(), values.data(), nullptr));
    return csr_dict(n, off, cols, values);
}

// homogeneous-Dirichlet Poisson solve (module.cpp:134-157): assemble
// (physics.cpp:10-75), condense the boundary nodes (solver.cpp:34-85),
// Jacobi BiCGSTAB (solver.cpp:105-227), expand
py::dict solve_poisson(Mesh& mesh, py::object diffusion, double source) {
    tgk_mesh* m = mesh.device();
    tgk_routing* r = mesh.routing();
    tgk_routing_view v{};
    check(tgk_routing_get_view(r, &v));
    const int64_t E = mesh.element_count(), N = v.N;
    tgk_problem p{};
    p.kind = TGK_POISSON;
    p.mode = TGK_MODE_EXACT;
    p.diffusion = tgk_field{TGK_FIELD_CONSTANT, 1.0, nullptr, 0};
    std::unique_ptr<DevBuf> drho;
    if (!diffusion.is_none()) {
        const auto rho = from_array(diffusion.cast<py::array_t<double, py::array::c_style | py::array::forcecast>>());
        drho = std::make_unique<DevBuf>(rho.data(), rho.size() * sizeof(double));
        p.diffusion = tgk_field{TGK_FIELD_ELEMENT, 0.0, drho->as<double>(), static_cast<int64_t>(rho.size())};
    }
    (void)E;
    p.n_source = 1;
    p.source[0] = tgk_field{TGK_FIELD_CONSTANT, source, nullptr, 0};
    DevBuf dK(static_cast<size_t>(v.nnz) * sizeof(double)), dF(static_cast<size_t>(N) * sizeof(double));
    check(tgk_assemble_d(&p, m, r, dK.as<double>(), dF.as<double>(), nullptr, nullptr));
    const auto& b = mesh.boundary_nodes();
    const std::vector<double> zeros(b.size(), 0.0);
    DevBuf ddofs(b.data(), b.size() * sizeof(int64_t)), dvals(zeros.data(), zeros.size() * sizeof(double));
    tgk_condensed* c = nullptr;
    check(tgk_condense_d(N, v.row_ptr, v.col_idx, dK.as<double>(), dF.as<double>(), static_cast<int64_t>(b.size()),
                         ddofs.as<int64_t>(), dvals.as<double>(), nullptr, &c));
    std::unique_ptr<tgk_condensed, void (*)(tgk_condensed*)> guard(c, tgk_condensed_destroy);
    int64_t nf = 0, nc = 0, nz = 0;
    const int64_t *d_off = nullptr, *d_cols = nullptr;
    const double *d_vals = nullptr, *d_Ff = nullptr;
    check(tgk_condensed_info(c, &nf, &nc, &nz, nullptr, nullptr, nullptr, &d_off, &d_cols, &d_vals, &d_Ff));
    DevBuf du(static_cast<size_t>(N) * sizeof(double));
    int64_t iters = 0;
    double rel = 0.0;
    if (nf > 0) {
        std::vector<double> x0(static_cast<size_t>(nf), 0.0);
        DevBuf dx(x0.data(), x0.size() * sizeof(double));
        int converged = 0;
        check(tgk_bicgstab_d(nf, d_off, d_cols, d_vals, d_Ff, dx.as<double>(), 1e-10, 1e-10, 10000, &iters, &rel,
                             &converged, nullptr));
        if (!converged)
            throw NumericalError("linear solve did not converge: rel_residual = " + std::to_string(rel) + " after " +
                                 std::to_string(iters) + " iterations");
        check(tgk_expand_d(c, dx.as<double>(), du.as<double>(), nullptr));
    } else {
        check(tgk_expand_d(c, nullptr, du.as<double>(), nullptr));
    }
    std::vector<double> u(static_cast<size_t>(N));
    du.to_host(u.data(), u.size());
    py::dict d;
    d["u"] = to_array(u);
    d["iterations"] = iters;
    d["rel_residual"] = rel;
    return d;
}

// compliance C = F^T U (adjoint.cpp:96-99), serial left fold
double compliance(const py::array_t<double, py::array::c_style | py::array::forcecast>& F,
                  const py::array_t<double, py::array::c_style | py::array::forcecast>& U) {
    if (F.size() != U.size()) throw InputError("compliance: size mismatch");
    double s = 0.0;
    for (py::ssize_t i = 0; i < F.size(); ++i) s += F.data()[i] * U.data()[i];
    return s;
}

std::shared_ptr<Mesh> from_python_mesh(py::object pm) {
    const int code = kind_code(pm.attr("kind").cast<std::string>());
    auto nodes = from_array(pm.attr("nodes").cast<py::array_t<double, py::array::c_style | py::array::forcecast>>());
    auto el = pm.attr("elements").cast<py::array_t<int64_t, py::array::c_style | py::array::forcecast>>();
    std::vector<int64_t> elems(el.data(), el.data() + el.size());
    auto bn = pm.attr("boundary_nodes").cast<py::array_t<int64_t, py::array::c_style | py::array::forcecast>>();
    std::vector<int64_t> boundary(bn.data(), bn.data() + bn.size());
    return std::make_shared<Mesh>(code, std::move(nodes), std::move(elems), std::move(boundary));
}

}  // namespace

PYBIND11_MODULE(_tgfem, m) {
    m.doc() = "tensorized map-reduce Galerkin assembly (B200 / libtgk)";
    py::register_exception<InputError>(m, "InputError");
    py::register_exception<NumericalError>(m, "NumericalError");

    py::class_<Mesh, std::shared_ptr<Mesh>>(m, "Mesh")
        .def_property_readonly("kind", [](const Mesh& mm) { return std::string(kind_name(mm.kind())); })
        .def_property_readonly("dim", &Mesh::dim)
        .def_property_readonly("nodes",
                               [](const Mesh& mm) { return to_array(mm.nodes()).reshape({mm.node_count(), int64_t(mm.dim())}); })
        .def_property_readonly("elements",
                               [](const Mesh& mm) { return to_array(mm.elements()).reshape({mm.element_count(), int64_t(mm.k())}); })
        .def_property_readonly("boundary_nodes", [](Mesh& mm) { return to_array(mm.boundary_nodes()); })
        .def("node_count", &Mesh::node_count)
        .def("element_count", &Mesh::element_count)
        .def("content_hash", &Mesh::content_hash);

    m.def("generate_grid", &make_grid, py::arg("kind"), py::arg("extents"), py::arg("divisions"));
    m.def("load_gmsh",
          [](const std::string& path) {
              return from_python_mesh(py::module_::import("paper_2602_05052_b200.tgfem").attr("load_gmsh")(path));
          },
          py::arg("path"));
    m.def("write_gmsh",
          [](Mesh& mesh, const std::string& path) {
              auto tg = py::module_::import("paper_2602_05052_b200.tgfem");
              py::object pm = tg.attr("Mesh")(kind_name(mesh.kind()),
                                              to_array(mesh.nodes()).reshape({mesh.node_count(), int64_t(mesh.dim())}),
                                              to_array(mesh.elements()).reshape({mesh.element_count(), int64_t(mesh.k())}),
                                              to_array(mesh.boundary_nodes()));
              tg.attr("write_gmsh")(pm, path);
          },
          py::arg("mesh"), py::arg("path"));
    m.def("set_thread_count", [](int n) { tgk_set_thread_count(n); }, py::arg("n"));
    m.def("local_stiffness", &local_stiffness, py::arg("mesh"), py::arg("coeff") = py::none(),
          "batched diffusion stiffness blocks, E x k x k");
    m.def("reduce_matrix", &reduce_matrix, py::arg("mesh"), py::arg("local_matrices"));
    m.def("scatter_add_oracle", &scatter_add_oracle, py::arg("mesh"), py::arg("local_matrices"));
    m.def("solve_poisson", &solve_poisson, py::arg("mesh"), py::arg("diffusion") = py::none(), py::arg("source") = 1.0,
          "homogeneous-Dirichlet Poisson solve; returns nodal solution");
    m.def("compliance", &compliance, py::arg("F"), py::arg("U"));
    m.def(
        "topopt_cantilever",
        [](int64_t, int64_t, int, double) -> py::dict {
            PyErr_SetString(PyExc_NotImplementedError,
                            "topopt_cantilever: SIMP topology optimisation on QUAD4 is outside the accelerated path");
            throw py::error_already_set();
        },
        py::arg("nx") = 60, py::arg("ny") = 30, py::arg("iterations") = 51, py::arg("vol_frac") = 0.5);
}
