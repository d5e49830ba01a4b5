// Host setup: assembled operators, interface alignment, subdomains and local
// operators -- the index-set machinery around the solve path.
//
// Restates (bit-exactly; the tests compare against the reference built in
// oracle/_ref byte for byte):
//   build_extension           proj/include/cpdd/operators.hpp:30-51
//   assemble_helmholtz        proj/include/cpdd/operators.hpp:79-112
//   SparseOperator::append_row proj/include/cpdd/sparse.hpp:33-49
//   align_interfaces          proj/include/cpdd/partition.hpp:474-508
//   load_partition checks     proj/include/cpdd/partition.hpp:519-552
//   find_cross_points         proj/include/cpdd/subdomain.hpp:59-79
//   build_subdomains          proj/include/cpdd/subdomain.hpp:153-313
//   assemble_local            proj/include/cpdd/transmission.hpp:73-138
// Work that the reference does serially (global rows, per-subdomain sets,
// local assembly) runs on a host thread pool here; every result is
// independent of the thread count.
#pragma once

#include "band.hpp"

#include <cstdint>
#include <functional>
#include <utility>
#include <vector>

namespace cpddg {

/** Row-compressed matrix with the reference's row-building rule. */
struct Csr {
    int rows = 0, cols = 0;
    std::vector<std::int64_t> ptr{0};
    std::vector<int> col;
    std::vector<double> val;
    std::int64_t nnz() const { return static_cast<std::int64_t>(col.size()); }
    /** sparse.hpp:33-49: sort scratch by column (std::sort, as the reference,
     *  so duplicate columns are summed in the same order), merge duplicates. */
    void append_row(std::vector<std::pair<int, double>>& scratch);
};

/** Run f(i, worker) for i in 0..n-1 on a transient pool of `workers`
 *  threads (0 = all hardware threads); worker ids are 0..workers-1. */
void parallel_for(int n, int workers, const std::function<void(int, int)>& f);
int resolve_workers(int workers);

template <int D>
Csr build_extension(const Band<D>& g, int workers = 0);

template <int D>
Csr assemble_helmholtz(const Band<D>& g, const Csr& E, double c, int workers = 0);

/** load_partition's validation (count, non-negative, no gaps); returns N_S. */
int validate_partition(const std::vector<int>& part, int n_active);

template <int D>
int align_interfaces(const Band<D>& g, std::vector<int>& part, int interp_degree);

template <int D>
std::vector<int> find_cross_points(const Band<D>& g, const std::vector<int>& part);

template <int D>
struct BoundaryNode {
    Ix<D> ix{};
    Vec<D> x{};
    bool is_ghost_type = false;
    int global_active = -1;
    Vec<D> cp{}, cp_local{}, conormal{};
    double dq = 0.0;
    bool cross_flagged = false;
    bool fallback = false;
};

template <int D>
struct Subdomain {
    int id = 0;
    std::vector<int> disjoint, overlap, final_layer, ghosts;
    std::vector<BoundaryNode<D>> bc;
    int fallback_count = 0;
    int n_lambda = 0;
};

template <int D>
std::vector<Subdomain<D>> build_subdomains(const Band<D>& g, const Surface<D>& surface,
                                           const std::vector<int>& part, const Csr& E,
                                           int n_overlap, bool robin_ring, int workers = 0);

struct TransmissionSpec {
    bool robin = true;
    double alpha = 1.0;
    double alpha_cross = 1.0;
};

/** LocalOperator (transmission.hpp:47-70) without the factorization: the
 *  factorization happens on the device (include/cpddg.h, cpddg_pc_create). */
struct LocalSystem {
    int id = 0;
    int n_overlap = 0, n_bc = 0;
    std::vector<int> overlap;
    std::vector<int> scatter_local, scatter_global;
    Csr A;
    int n_local() const { return n_overlap + n_bc; }
};

template <int D>
LocalSystem assemble_local(const Band<D>& g, const Csr& A, const Subdomain<D>& S,
                           const TransmissionSpec& spec, std::vector<int>& colmap_scratch);

template <int D>
std::vector<LocalSystem> assemble_locals(const Band<D>& g, const Csr& A,
                                         const std::vector<Subdomain<D>>& subs,
                                         const TransmissionSpec& spec, int workers = 0);

}  // namespace cpddg
