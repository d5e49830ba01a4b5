// Device setup entry points (csrc/cuda/setup_dev.cu), callable from the host
// setup: the band with its closest points, and the interface alignment and
// subdomain index sets, built on the GPU and bit-identical to the host
// restatement (band.cpp, decomp.cpp).
#pragma once

#include "decomp.hpp"

#include <memory>

namespace cpddg {

struct DevBand;  // device band of a setup (setup_dev.cuh)

/** Thrown by decompose_device when the problem exceeds its index packing
 *  (the caller then runs the host restatement). */
struct DeviceSetLimit : ConfigError {
    using ConfigError::ConfigError;
};

/** build_band_tube (band.hpp:150-182) on the device; the host copy is
 *  returned (with its lattice map), the device band kept in *keep. */
template <int D>
Band<D> build_band_device(const Surface<D>& surface, double h, int p, double tube_radius,
                          std::shared_ptr<DevBand>* keep);

/** align_interfaces (partition.hpp:474-508) and build_subdomains
 *  (subdomain.hpp:153-313) on the device for the band of `dev` (g is its host
 *  copy); part is aligned in place; returns the move count. */
template <int D>
int decompose_device(const DevBand& dev, const Band<D>& g, std::vector<int>& part, int n_overlap, bool robin_ring,
                     std::vector<Subdomain<D>>& subs, double* t_align, double* t_sets);

}  // namespace cpddg
