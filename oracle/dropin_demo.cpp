// ORACLE TEST INFRASTRUCTURE -- the drop-in demonstration.
//
// A reference caller's program, unchanged except for include/cpddg.hpp: the
// reference pipeline (RunConfig -> build_problem -> partition file ->
// align_interfaces -> build_subdomains -> assemble_local; pipeline.hpp:155-216,
// all from /root/reference/proj/include) feeds both the reference's CPU
// gmres_solve and the device gmres_solve overload from cpddg.hpp.  Prints one
// JSON line per case; tests/test_gpu_dropin.py checks them.
#include "cpdd/cpdd.hpp"
#include "cpddg.hpp"

#include <cmath>
#include <cstdio>
#include <fstream>

using namespace cpdd;

template <int D>
int run_case(const char* name, RunConfig cfg, int n_parts) {
    BuiltProblem<D> P = build_problem<D>(cfg);
    const int na = P.grid.n_active();
    // BASELINE partitions: sectors (2D) / a simple deterministic slab split (3D) -- written as a
    // partition file and loaded through the reference's load_partition
    std::vector<int> part(static_cast<std::size_t>(na));
    for (int i = 0; i < na; ++i) {
        const auto& cp = P.grid.active[static_cast<std::size_t>(i)].cp.cp;
        double t = std::atan2(cp[1], cp[0]);
        if (t < 0) t += 2 * M_PI;
        part[static_cast<std::size_t>(i)] = std::min(n_parts - 1, static_cast<int>(std::floor(n_parts * t / (2 * M_PI))));
    }
    const std::string path = std::string("/tmp/dropin_part_") + name + ".txt";
    save_partition(path, part);
    part = load_partition(path, na);
    align_interfaces(P.grid, part, P.grid.p);
    const SolverConfig& sc = cfg.solver;
    auto subs = build_subdomains(P.grid, P.surface, part, P.E, sc.n_overlap, sc.robin());
    TransmissionSpec spec;
    spec.kind = sc.robin() ? TransmissionSpec::Kind::robin : TransmissionSpec::Kind::dirichlet;
    spec.alpha = sc.alpha;
    spec.alpha_cross = sc.effective_alpha_cross();
    std::vector<LocalOperator> cpu_locals, dev_locals;
    for (const auto& S : subs) {
        cpu_locals.push_back(assemble_local(P.grid, P.A, S, spec, true));
        dev_locals.push_back(assemble_local(P.grid, P.A, S, spec, false));
    }
    SchwarzPreconditioner M(std::move(cpu_locals), na, nullptr);
    SolveResult ref = gmres_solve(P.A, P.b, &M, sc.rel_tol, 2000, sc.gmres_restart);

    DeviceHelmholtz dA(P.grid, sc.c);
    DeviceSchwarz dM(dev_locals, na);
    SolveResult dev = gmres_solve(dA, P.b, &dM, sc.rel_tol, 2000, sc.gmres_restart);
    const Eigen::VectorXd Ax = P.A.apply(P.b), dAx = dA.apply(P.b);
    const double op_err = (Ax - dAx).norm() / Ax.norm();
    const double u_err = (ref.u - dev.u).norm() / ref.u.norm();
    std::printf("{\"case\": \"%s\", \"n_active\": %d, \"ref_iters\": %d, \"dev_iters\": %d, \"ref_conv\": %d, "
                "\"dev_conv\": %d, \"u_rel_diff\": %.3e, \"op_rel_diff\": %.3e, \"dev_final_true\": %.6e, "
                "\"ref_final_true\": %.6e}\n",
                name, na, ref.log.iterations, dev.log.iterations, ref.log.converged, dev.log.converged, u_err, op_err,
                dev.log.final_true_residual, ref.log.final_true_residual);
    // error behaviour crosses the boundary as the reference exceptions
    try {
        DeviceHelmholtz bad(P.grid, -1.0);
        std::printf("{\"case\": \"%s_error\", \"raised\": 0}\n", name);
    } catch (const ConfigError&) {
        std::printf("{\"case\": \"%s_error\", \"raised\": 1}\n", name);
    }
    return 0;
}

int main() {
    RunConfig c2;
    c2.surface = "circle";
    c2.h = 0.0125;
    c2.p = 3;
    c2.rhs = "circle-harmonic";
    c2.harmonic = 12;
    c2.solver.method = SolverConfig::Method::oras;
    c2.solver.mode = SolverConfig::Mode::gmres;
    c2.solver.gmres_restart = 50;
    c2.solver.rel_tol = 1e-10;
    c2.solver.n_overlap = 2;
    c2.solver.n_subdomains = 8;
    run_case<2>("circle_oras", c2, 8);
    RunConfig c3;
    c3.surface = "sphere";
    c3.h = 0.05;
    c3.p = 3;
    c3.rhs = "sphere-field";
    c3.solver.method = SolverConfig::Method::oras;
    c3.solver.mode = SolverConfig::Mode::gmres;
    c3.solver.gmres_restart = 50;
    c3.solver.rel_tol = 1e-10;
    c3.solver.n_overlap = 2;
    c3.solver.alpha = 4.0;
    c3.solver.alpha_cross = 40.0;
    c3.solver.n_subdomains = 16;
    run_case<3>("sphere_oras_modified", c3, 16);
    return 0;
}
