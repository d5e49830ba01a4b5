// Internal definition of the cpddg_setup handle and the error plumbing
// shared by every C-ABI translation unit.
#pragma once

#include "../../../include/cpddg.h"
#include "decomp.hpp"
#include "setup_dev.hpp"

#include <memory>
#include <string>

struct cpddg_setup {
    int dim = 0;
    int workers = 0;
    int device_setup = 0;
    double c = 1.0;
    std::unique_ptr<void, void (*)(void*)> impl{nullptr, [](void*) {}};
};

namespace cpddg {

template <int D>
struct SetupImpl {
    Surface<D> surface;
    Band<D> band;
    Csr E, A;
    std::vector<int> part;
    int moves = 0;
    bool robin = false;
    std::vector<Subdomain<D>> subs;
    std::vector<LocalSystem> locals;
    std::shared_ptr<DevBand> dev;  // device band (device_setup)
    double t_band = 0, t_E = 0, t_A = 0, t_align = 0, t_sets = 0, t_local = 0;  // phase seconds
};

template <int D>
inline SetupImpl<D>& impl_of(const cpddg_setup* s) {
    if (!s || s->dim != D || !s->impl) throw InternalError("invalid setup handle");
    return *static_cast<SetupImpl<D>*>(s->impl.get());
}

/** Record msg as the calling thread's last error and return code. */
int set_error(int code, const std::string& msg);

/** Run f, mapping exceptions to status codes (include/cpddg.h). */
template <class F>
int guarded(F&& f) {
    try {
        f();
        return CPDDG_OK;
    } catch (const ConfigError& e) {
        return set_error(CPDDG_ERR_CONFIG, std::string("ConfigError: ") + e.what());
    } catch (const DivergenceError& e) {
        return set_error(CPDDG_ERR_DIVERGENCE, std::string("DivergenceError: ") + e.what());
    } catch (const IoError& e) {
        return set_error(CPDDG_ERR_IO, std::string("IoError: ") + e.what());
    } catch (const InternalError& e) {
        return set_error(CPDDG_ERR_INTERNAL, std::string("InternalError: ") + e.what());
    } catch (const std::bad_alloc&) {
        return set_error(CPDDG_ERR_INTERNAL, "InternalError: host allocation failed");
    } catch (const std::exception& e) {
        const std::string w = e.what();
        if (w.rfind("CUDA", 0) == 0) return set_error(CPDDG_ERR_CUDA, w);
        return set_error(CPDDG_ERR_INTERNAL, std::string("InternalError: ") + w);
    }
}

}  // namespace cpddg
