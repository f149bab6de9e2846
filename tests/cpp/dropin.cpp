// dropin.cpp — a consumer written against the reference's C++ API (namespace sparsla,
// reference sparse.hpp / errors.hpp names) compiled against include/sparsla/*.hpp and
// linked to libsparsla_b200.so.  Mode "cpu": host-only parts; mode "gpu": solves on cuda:0.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>

#include "sparsla/adjoint.hpp"
#include "sparsla/distributed.hpp"
#include "sparsla/eigen.hpp"
#include "sparsla/solve.hpp"
#include "sparsla/sparse.hpp"

using namespace sparsla;

#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)

static SparseCoo poisson2d(index_t N) {
    std::vector<index_t> r, c;
    std::vector<double> v;
    for (index_t i = 0; i < N; ++i)
        for (index_t j = 0; j < N; ++j) {
            const index_t k = i * N + j;
            // emitted in reverse to exercise canonicalization
            if (i < N - 1) { r.push_back(k); c.push_back(k + N); v.push_back(-1.0); }
            if (j < N - 1) { r.push_back(k); c.push_back(k + 1); v.push_back(-1.0); }
            r.push_back(k); c.push_back(k); v.push_back(2.5);
            r.push_back(k); c.push_back(k); v.push_back(1.5);  // duplicate: summed to 4
            if (j > 0) { r.push_back(k); c.push_back(k - 1); v.push_back(-1.0); }
            if (i > 0) { r.push_back(k); c.push_back(k - N); v.push_back(-1.0); }
        }
    return SparseCoo(r, c, v, Shape{N * N, N * N});
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    // --- host-side API (sparse.hpp) ---
    SparseCoo a({0, 0}, {0, 0}, {1.0, 2.0}, Shape{1, 1});
    CHECK(a.nnz() == 1 && a.vals()[0] == 3.0);
    bool threw = false;
    try { SparseCoo bad({0}, {3}, {1.0}, Shape{2, 2}); } catch (const BoundsError&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { SparseCoo bad({0, 1}, {0}, {1.0}, Shape{2, 2}); } catch (const DimensionError&) { threw = true; }
    CHECK(threw);
    SparseCoo P = poisson2d(16);
    CHECK(P.nnz() == 5 * 256 - 4 * 16);
    CHECK(P.find(0, 0) == 0 && P.vals()[0] == 4.0 && P.find(0, 2) == -1);
    CsrMatrix A = CsrMatrix::from_coo(P);
    CHECK(A.row_ptr()[256] == P.nnz() && A.bytes() == (257 + 2 * P.nnz()) * 8);
    SparseCoo back = A.to_coo();
    CHECK(back.nnz() == P.nnz() && back.rows()[5] == P.rows()[5]);
    CHECK(is_symmetric(P) && is_structurally_symmetric(P));
    SparseCoo T = transpose(SparseCoo({0}, {1}, {1.0}, Shape{2, 3}));
    CHECK(T.nrows() == 3 && T.rows()[0] == 1 && T.cols()[0] == 0);
    auto part = partition_contiguous(6, 2);
    CHECK(part[2] == 0 && part[3] == 1);
    threw = false;
    try { partition_contiguous(3, 4); } catch (const InvalidArgumentError&) { threw = true; }
    CHECK(threw);
    std::vector<index_t> owned = {0, 1, 2};
    SparseCoo chain({0, 0, 1, 1, 1, 2, 2, 2}, {0, 1, 0, 1, 2, 1, 2, 3}, {2, -1, -1, 2, -1, -1, 2, -1}, Shape{3, 6});
    LocalPartition L(6, &part, 2, 0, owned, CsrMatrix::from_coo(chain));
    CHECK(L.halo().size() == 1 && L.halo()[0] == 3 && L.send_idx()[0] == 2 && L.recv_idx()[0] == 3);
    // SPEC build_local(A: SparseCoo, part_of, rank) on the Figure-1 chain
    SparseCoo chain6({0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3, 4, 4, 4, 5, 5},
                     {0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4, 5, 4, 5},
                     {2, -1, -1, 2, -1, -1, 2, -1, -1, 2, -1, -1, 2, -1, -1, 2}, Shape{6, 6});
    LocalPartition L0 = build_local(chain6, part, 0), L1 = build_local(chain6, part, 1);
    CHECK(L0.owned().size() == 3 && L0.halo().size() == 1 && L0.halo()[0] == 3 && L0.neighbors()[0] == 1);
    CHECK(L1.halo().size() == 1 && L1.halo()[0] == 2 && L1.send_idx()[0] == 0);
    if (!gpu) { std::printf("dropin cpu ok\n"); return 0; }
    // --- GPU path ---
    std::vector<double> ones(256, 1.0);
    auto y = spmv(A, ones);
    CHECK(y[0] == 2.0 && y[17] == 0.0);
    auto [x, rep] = cg_solve(A, ones, SolveOptions{});
    CHECK(rep.converged && rep.residual_norm <= 1e-10 && rep.spmv_count == rep.iterations + 1);
    auto r = spmv(A, x);
    double err = 0;
    for (int i = 0; i < 256; ++i) err = std::fmax(err, std::fabs(r[i] - 1.0));
    CHECK(err < 1e-9);
    auto [xb, repb] = bicgstab_solve(A, ones, SolveOptions{1e-12, 0.0, 1000, Preconditioner::jacobi});
    CHECK(repb.converged && repb.backend == Backend::bicgstab);
    auto d = jacobi_build(A);
    CHECK(d.inverse_diagonal[3] == 0.25);
    SparseCoo I2({0, 1, 2}, {0, 1, 2}, {2.0, 2.0, 2.0}, Shape{3, 3});
    std::vector<double> b3 = {2, 4, 6}, g3 = {1, 1, 1};
    auto [x3, ctx] = solve_forward(I2, b3);
    auto grads = solve_backward(ctx, g3);
    CHECK(grads.grad_b[0] == 0.5 && grads.grad_vals[2] == -1.5);
    // eigen-solver: [[2,1],[1,2]], k = 1 -> lambda = 1, dlambda/dA = v v^T
    SparseCoo E({0, 0, 1, 1}, {0, 1, 0, 1}, {2.0, 1.0, 1.0, 2.0}, Shape{2, 2});
    auto ev = eig_smallest(E, 1, 1e-10);
    CHECK(std::fabs(ev.lambdas[0] - 1.0) < 1e-14 && ev.vectors[0] > 0 && ev.report.converged);
    std::vector<double> gl = {1.0};
    auto ge = eig_backward(ev, E, gl);
    CHECK(std::fabs(ge[0] - 0.5) < 1e-14 && std::fabs(ge[1] + 0.5) < 1e-14);
    auto ep = eig_smallest(P, 6, 1e-9);  // 2-D Poisson 16x16 through LOBPCG
    CHECK(ep.report.converged && std::fabs(ep.lambdas[0] - 2.0 * (2.0 - 2.0 * std::cos(M_PI / 17))) < 1e-8);
    // --- SPEC-shaped distributed API: 2 in-process ranks on cuda:0 ---
    {
        const auto pc = partition_contiguous(256, 2);
        const auto [xs, rs] = cg_solve(A, ones, SolveOptions{});
        const auto ys = spmv(A, xs);
        LocalHub hub(2);
        int fails[2] = {0, 0};
        auto worker = [&](int rank) {
            try {
                Transport T = Transport::in_process(hub, rank, 0);
                LocalPartition L = build_local(P, pc, rank);
                const auto& own = L.owned();
                std::vector<double> xo(own.size());
                for (std::size_t i = 0; i < own.size(); ++i) xo[i] = xs[own[i]];
                auto halo = halo_exchange(L, T, xo);
                for (std::size_t i = 0; i < halo.size(); ++i) fails[rank] += halo[i] != xs[L.halo()[i]];
                auto yo = dist_spmv(L, T, xo);
                for (std::size_t i = 0; i < own.size(); ++i) fails[rank] += yo[i] != ys[own[i]];
                fails[rank] += all_reduce_sum(T, rank + 1.0) != 3.0;
                std::vector<double> bo(own.size(), 1.0);
                auto [xd, rd] = dist_cg(L, T, bo, 1e-10, 10000);
                fails[rank] += !rd.converged || rd.iterations != rs.iterations;
                double e = 0;
                for (std::size_t i = 0; i < own.size(); ++i) e = std::fmax(e, std::fabs(xd[i] - xs[own[i]]));
                fails[rank] += e > 1e-10;
                auto g = dist_adjoint_solve(L, T, xd, bo);
                fails[rank] += !g.report.converged || g.grad_b_owned.size() != own.size();
                for (std::size_t i = 0; i < own.size(); ++i) fails[rank] += std::fabs(g.grad_b_owned[i] - xd[i]) > 1e-12;
                auto xg = gather_solution(L, T, xd);
                if (rank == 0) {
                    fails[rank] += xg.size() != 256;
                    for (std::size_t i = 0; i < xg.size(); ++i) fails[rank] += std::fabs(xg[i] - xs[i]) > 1e-10;
                } else {
                    fails[rank] += !xg.empty();
                }
                fails[rank] += T.all_reduces() <= 0;
            } catch (const std::exception& ex) {
                std::printf("rank %d: %s\n", rank, ex.what());
                fails[rank] += 1000;
            }
        };
        std::thread t0(worker, 0), t1(worker, 1);
        t0.join();
        t1.join();
        CHECK(fails[0] == 0 && fails[1] == 0);
    }
    std::printf("dropin gpu ok\n");
    return 0;
}
