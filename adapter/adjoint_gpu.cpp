// GPU drop-in for tg::simp_sensitivity (proj/include/tg/adjoint.hpp:37-42,
// proj/src/adjoint.cpp:101-125): dC/drho_e = -p rho_e^{p-1} (E_max - E_min)
// u_e^T K0_e u_e for any element kind and DoF map (the topology-optimisation
// loop's vector-elasticity sensitivity, topopt.cpp), computed by libtgk's
// tgk_simp_sensitivity_d through its C ABI.  Compiled against the UNMODIFIED
// reference headers; linked in place of adjoint.cpp's function (oracle/Makefile
// renames the reference symbol with objcopy, like tg::assemble).
//
// Contract kept from the reference: the same shape check and InputError
// message (adjoint.cpp:107-110); values bit-identical for the standard penalty
// p = 3 (the reference's operation order, libtgk compiled without FMA
// contraction), within one ulp of std::pow otherwise.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tg/adjoint.hpp"
#include "tg/errors.hpp"
#include "tgk.h"

namespace tg {

namespace {

[[noreturn]] void raise_adj(int rc) {
    const std::string msg = tgk_last_error();
    if (rc == TGK_ERR_INPUT) throw InputError(msg);
    if (rc == TGK_ERR_NUMERICAL) throw NumericalError(msg);
    throw std::runtime_error("libtgk: " + msg);
}

void check_adj(int rc) {
    if (rc != TGK_OK) raise_adj(rc);
}

// device copy of a host vector, freed on scope exit
struct DeviceCopy {
    void* p = nullptr;
    DeviceCopy(const void* host, std::size_t bytes) {
        check_adj(tgk_alloc_d(&p, static_cast<std::int64_t>(bytes)));
        if (bytes) check_adj(tgk_copy_h2d(p, host, static_cast<std::int64_t>(bytes)));
    }
    explicit DeviceCopy(std::size_t bytes) { check_adj(tgk_alloc_d(&p, static_cast<std::int64_t>(bytes))); }
    ~DeviceCopy() { tgk_free_d(p); }
    DeviceCopy(const DeviceCopy&) = delete;
    DeviceCopy& operator=(const DeviceCopy&) = delete;
};

}  // namespace

std::vector<double> simp_sensitivity(const std::vector<double>& rho, double p, double E_min, double E_max,
                                     const std::vector<double>& unit_stiffness, const Mesh& mesh,
                                     const DofMap& dofmap, const std::vector<double>& U) {
    const std::int64_t E = mesh.element_count();
    const int k = dofmap.k;
    if (static_cast<std::int64_t>(rho.size()) != E ||
        unit_stiffness.size() != static_cast<std::size_t>(E) * k * k)
        throw InputError("simp_sensitivity: shape mismatch");  // adjoint.cpp:107-110
    std::vector<double> sens(static_cast<std::size_t>(E));
    if (E == 0) return sens;
    DeviceCopy d_map(dofmap.map.data(), dofmap.map.size() * sizeof(std::int64_t));
    DeviceCopy d_rho(rho.data(), rho.size() * sizeof(double));
    DeviceCopy d_k0(unit_stiffness.data(), unit_stiffness.size() * sizeof(double));
    DeviceCopy d_u(U.data(), U.size() * sizeof(double));
    DeviceCopy d_out(sens.size() * sizeof(double));
    check_adj(tgk_simp_sensitivity_d(E, k, static_cast<const std::int64_t*>(d_map.p), static_cast<const double*>(d_rho.p),
                                     p, E_min, E_max, static_cast<const double*>(d_k0.p),
                                     static_cast<const double*>(d_u.p), static_cast<std::int64_t>(U.size()),
                                     static_cast<double*>(d_out.p), nullptr));
    check_adj(tgk_copy_d2h(sens.data(), d_out.p, static_cast<std::int64_t>(sens.size() * sizeof(double))));
    return sens;
}

}  // namespace tg
