// extern "C" boundary of libsgw_b200.so (declared in include/sgw.h).
// Host buffers in, host buffers out; exceptions become sgw_status codes.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/sgw.h"
#include "generic.cuh"
#include "solver.cuh"

using namespace sgw;

struct sgw_solver {
  std::unique_ptr<GpuSolver> g;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SGW_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return SGW_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SGW_EINVAL;
  }
}

struct Tmp {  // device scratch for host<->device copies
  DBuf<double> a, b;
};

void h2d(DBuf<double>& d, const double* h, size_t n, cudaStream_t st) {
  if (d.n < n) d.alloc(n);
  SGW_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(double), cudaMemcpyHostToDevice, st));
}
void d2h(double* h, const double* d, size_t n, cudaStream_t st) {
  SGW_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  SGW_CUDA(cudaStreamSynchronize(st));
}

void set_force(GpuSolver& g, const sgw_force* f, int rows) {
  if (!f || f->kind == 0) {
    g.set_force_point(-1, 0, 0, 0);
  } else if (f->kind == 1) {
    if (f->node < 0 || f->node >= g.P.n_nodes()) throw Error(SGW_EINVAL, "force node out of range");
    g.set_force_point(f->node, f->f0, f->t0, f->amp);
  } else if (f->kind == 2) {
    if (!f->table || rows < 1) throw Error(SGW_EINVAL, "force table needs sgw_run (rows = n_steps + 1)");
    g.set_force_table(f->table, rows);
  } else {
    throw Error(SGW_EINVAL, "unknown force kind");
  }
}
// global interface vectors in and out (every rank passes and gets the whole vector)
template <typename F>
void iface_op(GpuSolver& g, const double* x, double* y, F&& op) {
  if (g.NGG == 0) return;  // one subdomain: the interface system is empty
  DBuf<double> gx, lx, ly, gy;
  h2d(gx, x, g.NGG, g.stream());
  lx.alloc(g.NG), ly.alloc(g.NG), gy.alloc(g.NGG);
  g.iface_to_local(gx.p, lx.p);
  op(lx.p, ly.p);
  g.iface_to_global(ly.p, gy.p);
  d2h(y, gy.p, g.NGG, g.stream());
}
}  // namespace

struct sgw_schur {
  std::unique_ptr<GenericSchur> g;
};

namespace {
template <typename F>
int gschur_apply(sgw_schur* h, const double* in, double* out, F&& f) {
  return guard([&] {
    GenericSchur& g = *h->g;
    const long long n = g.n_global();
    DBuf<double> a, b;
    a.alloc(std::max<long long>(1, n)), b.alloc(std::max<long long>(1, n));
    SGW_CUDA(cudaMemcpyAsync(a.p, in, n * 8, cudaMemcpyHostToDevice, g.stream()));
    f(g, a.p, b.p);
    SGW_CUDA(cudaMemcpyAsync(out, b.p, n * 8, cudaMemcpyDeviceToHost, g.stream()));
    SGW_CUDA(cudaStreamSynchronize(g.stream()));
  });
}
void report_out(int it, bool conv, const std::vector<double>& h, int* iterations, int* converged, double* hist,
                int hist_cap, int* hist_len) {
  if (iterations) *iterations = it;
  if (converged) *converged = conv ? 1 : 0;
  if (hist_len) *hist_len = (int)h.size();
  if (hist)
    for (int i = 0; i < std::min<int>(hist_cap, (int)h.size()); ++i) hist[i] = h[i];
}
}  // namespace

extern "C" {

const char* sgw_last_error(void) { return g_err.c_str(); }
int sgw_version(void) { return 1; }

namespace {
Problem problem_from(const sgw_problem* p) {
    if (!p) throw Error(SGW_EINVAL, "null argument");
    if (!p->coeff || p->n_input < 1) throw Error(SGW_EINVAL, "SgSolver: empty coefficient field");
    Problem P;
    P.nx = p->nx, P.ny = p->ny, P.px = p->px, P.py = p->py;
    P.n_in = p->n_input;
    P.nt = p->n_output;
    if (P.nx < 2 || P.ny < 2) throw Error(SGW_EINVAL, "build_unit_square_mesh: nx and ny must be >= 2");
    P.coeff.assign(p->coeff, p->coeff + (size_t)P.n_in * P.n_nodes());
    P.tensor.n_in = p->n_input;
    P.tensor.n_out = p->n_output;
    for (int e = 0; e < p->n_entries; ++e) {
      P.tensor.i.push_back(p->ent_i[e]);
      P.tensor.j.push_back(p->ent_j[e]);
      P.tensor.k.push_back(p->ent_k[e]);
      P.tensor.v.push_back(p->ent_v[e]);
    }
    P.density = p->density, P.alpha0 = p->alpha0, P.alpha1 = p->alpha1;
    P.gamma = p->gamma, P.zeta = p->zeta, P.dt = p->dt, P.tol = p->tol, P.max_iter = p->max_iter;
    P.device = p->device, P.rank = p->rank, P.world = p->world_size < 1 ? 1 : p->world_size;
    if (p->precond < 0 || p->precond > 2) throw Error(SGW_EINVAL, "unknown preconditioner");  // precond_from_string
    P.precond = p->precond;
    P.implicit_schur = p->implicit_schur != 0;
    if (P.rank < 0 || P.rank >= P.world) throw Error(SGW_EINVAL, "rank out of range");
    if (P.world > P.px * P.py) throw Error(SGW_EINVAL, "more ranks than subdomains");
    return P;
}
}  // namespace

int sgw_create(const sgw_problem* p, sgw_solver** out) {
  return guard([&] {
    if (!out) throw Error(SGW_EINVAL, "null argument");
    Problem P = problem_from(p);
    std::unique_ptr<Comm> comm;
    if (P.world > 1 && !p->nccl_id) throw Error(SGW_EINVAL, "world_size > 1 needs the NCCL unique id of rank 0");
    if (p->nccl_id) comm = make_nccl_comm(p->nccl_id, P.rank, P.world, P.device);  // also a 1-rank communicator
    auto s = std::make_unique<sgw_solver>();
    s->g = std::make_unique<GpuSolver>(std::move(P), std::move(comm));
    *out = s.release();
  });
}

int sgw_create_local_group(const sgw_problem* p, int world_size, int rank, void* group, sgw_solver** out) {
  return guard([&] {
    if (!out || !group) throw Error(SGW_EINVAL, "null argument");
    auto* g = static_cast<std::shared_ptr<ThreadGroup>*>(group);
    Problem P = problem_from(p);
    P.rank = rank, P.world = world_size;
    if (rank < 0 || rank >= world_size || world_size > P.px * P.py)
      throw Error(SGW_EINVAL, "rank / world_size out of range");
    auto s = std::make_unique<sgw_solver>();
    s->g = std::make_unique<GpuSolver>(std::move(P), make_thread_comm(*g, rank));
    *out = s.release();
  });
}

int sgw_create_solo(const sgw_problem* p, int world_size, int rank, sgw_solver** out) {
  return guard([&] {
    if (!out) throw Error(SGW_EINVAL, "null argument");
    Problem P = problem_from(p);
    P.rank = rank, P.world = world_size;
    if (rank < 0 || rank >= world_size || world_size > P.px * P.py)
      throw Error(SGW_EINVAL, "rank / world_size out of range");
    auto s = std::make_unique<sgw_solver>();
    s->g = std::make_unique<GpuSolver>(std::move(P), make_solo_comm(rank, world_size));
    *out = s.release();
  });
}

int sgw_local_group_new(int world_size, void** group) {
  return guard([&] {
    if (!group || world_size < 1) throw Error(SGW_EINVAL, "bad argument");
    *group = new std::shared_ptr<ThreadGroup>(make_thread_group(world_size));
  });
}

int sgw_local_group_abort(void* group) {
  return guard([&] { thread_group_abort(**static_cast<std::shared_ptr<ThreadGroup>*>(group)); });
}

int sgw_local_group_free(void* group) {
  return guard([&] { delete static_cast<std::shared_ptr<ThreadGroup>*>(group); });
}

int sgw_destroy(sgw_solver* s) {
  return guard([&] { delete s; });
}

int sgw_sizes(sgw_solver* s, long long* o) {
  return guard([&] {
    GpuSolver& g = *s->g;
    o[0] = g.n;
    o[1] = g.NT;
    o[2] = g.G.n_iface_global;
    o[3] = g.G.n_corner;
    o[4] = g.NGG;
    o[5] = g.G.ns_total;
    o[6] = 0;
    o[7] = g.device_bytes();
  });
}

int sgw_set_stream(sgw_solver* s, void* stream) {
  return guard([&] { s->g->set_stream(static_cast<cudaStream_t>(stream)); });
}

int sgw_apply_block(sgw_solver* s, int op, const double* x, double* y) {
  return guard([&] {
    GpuSolver& g = *s->g;
    if (op < 0 || op > 2) throw Error(SGW_EINVAL, "apply_block: op must be 0, 1 or 2");
    DBuf<double> dx, dy;
    h2d(dx, x, g.NSTATE, g.stream());
    dy.alloc(g.NSTATE);
    g.apply_block(op, dx.p, dy.p);
    d2h(y, dy.p, g.NSTATE, g.stream());
  });
}

int sgw_schur_matvec(sgw_solver* s, const double* x, double* y) {
  return guard([&] {
    GpuSolver& g = *s->g;
    iface_op(g, x, y, [&](const double* a, double* b) { g.schur_matvec(a, b); });
  });
}

int sgw_apply_nn2(sgw_solver* s, const double* r, double* z) {
  return guard([&] {
    GpuSolver& g = *s->g;
    iface_op(g, r, z, [&](const double* a, double* b) { g.apply_nn2(a, b); });
  });
}

int sgw_apply_precond(sgw_solver* s, int kind, const double* r, double* z) {
  return guard([&] {
    GpuSolver& g = *s->g;
    if (kind < 0 || kind > 2) throw Error(SGW_EINVAL, "unknown preconditioner");
    iface_op(g, r, z, [&](const double* a, double* b) { g.apply_precond(kind, a, b); });
  });
}

int sgw_pcg(sgw_solver* s, const double* rhs, double* x, int* iterations, int* converged, double* hist,
            int cap) {
  return guard([&] {
    GpuSolver& g = *s->g;
    bool conv = false;
    std::vector<double> h;
    int it = 0;
    iface_op(g, rhs, x, [&](const double* b, double* xx) { it = g.pcg(b, xx, &conv, &h); });
    if (iterations) *iterations = it;
    if (converged) *converged = conv ? 1 : 0;
    if (hist)
      for (int i = 0; i < cap; ++i) hist[i] = i < (int)h.size() ? h[i] : -1.0;
  });
}

int sgw_coarse_operator(sgw_solver* s, double* out) {
  return guard([&] {
    const auto f = s->g->coarse_operator_host();
    std::memcpy(out, f.data(), f.size() * sizeof(double));
  });
}

int sgw_local_block(sgw_solver* s, int sub, int which, double* out, long long* gmap, long long* dims) {
  return guard([&] {
    GpuSolver& g = *s->g;
    const int sl = g.local_sub(sub);
    if (sl < 0 || sl >= g.NS) throw Error(SGW_EINVAL, "subdomain is not owned by this rank");
    if (which < 0 || which > 2) throw Error(SGW_EINVAL, "which must be 0 (S), 1 (S_rr^-1) or 2 (Psi)");
    if (dims) g.local_dims(sl, dims);
    if (!out && !gmap) return;
    std::vector<long long> gm;
    const std::vector<double> v = g.local_block(sl, which, gmap ? &gm : nullptr);
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
    if (gmap) std::memcpy(gmap, gm.data(), gm.size() * sizeof(long long));
  });
}

int sgw_init_state(sgw_solver* s, const double* u0, const double* v0, const sgw_force* force) {
  return guard([&] {
    GpuSolver& g = *s->g;
    set_force(g, force, 0);
    h2d(g.nodal_u0_, u0, g.P.n_nodes(), g.stream());
    h2d(g.nodal_v0_, v0, g.P.n_nodes(), g.stream());
    g.init_state(g.nodal_u0_.p, g.nodal_v0_.p, 0.0);
  });
}

int sgw_advance(sgw_solver* s, int n_steps, int* iterations) {
  return guard([&] {
    GpuSolver& g = *s->g;
    for (int k = 0; k < n_steps; ++k) {
      int it = 0;
      g.step(&it, k + 1 < n_steps);
      if (iterations) iterations[k] = it;
    }
  });
}

int sgw_get_state(sgw_solver* s, double* u_flat) {
  return guard([&] {
    GpuSolver& g = *s->g;
    DBuf<double> full;
    full.alloc(g.NSTATE);
    g.gather_state(full.p);
    d2h(u_flat, full.p, g.NSTATE, g.stream());
  });
}

int sgw_run(sgw_solver* s, const double* u0, const double* v0, int n_steps, const sgw_force* force,
            sgw_history* h) {
  return guard([&] {
    GpuSolver& g = *s->g;
    if (n_steps < 0) throw Error(SGW_EINVAL, "n_steps must be >= 0");
    // probes (src/sg.cpp:378-383)
    g.probe_dofs.clear();
    const int np = h ? h->n_probes : 0;
    for (int p = 0; p < np; ++p) {
      const int node = h->probe_nodes[p];
      if (node < 0 || node >= g.P.n_nodes()) throw Error(SGW_EINVAL, "probe node out of range");
      const int gi = node % (g.P.nx + 1), gj = node / (g.P.nx + 1);
      const int d = g.G.dof(gi, gj);
      if (d < 0) throw Error(SGW_EINVAL, "probe node is constrained");
      g.probe_dofs.push_back(d);
    }
    g.probe_cap = n_steps + 1;
    if (np) {
      g.d_probe_dofs.upload(g.probe_dofs);
      std::vector<int> own(np);
      for (int q = 0; q < np; ++q) own[q] = g.G.owner_of_dof(g.probe_dofs[q]) == g.rank();
      g.d_probe_own.upload(own);
      const size_t need = (size_t)(n_steps + 1) * np * (2 + g.NT);
      if (g.probe_hist.n < need) g.probe_hist.alloc(need);
    }
    set_force(g, force, n_steps + 1);
    struct TableScope {  // a force table is the caller's memory: it is dropped when the run ends
      GpuSolver& g;
      ~TableScope() { g.drop_force_table(); }
    } table_scope{g};
    h2d(g.nodal_u0_, u0, g.P.n_nodes(), g.stream());
    h2d(g.nodal_v0_, v0, g.P.n_nodes(), g.stream());
    g.init_state(g.nodal_u0_.p, g.nodal_v0_.p, 0.0);
    g.record_probes(0);
    DBuf<double> full;
    if (h && h->full_state) {
      full.alloc(g.NSTATE);
      g.gather_state(full.p);
      d2h(h->full_state, full.p, g.NSTATE, g.stream());
    }
    for (int k = 0; k < n_steps; ++k) {
      int it = 0;
      g.step(&it, k + 1 < n_steps);
      if (h && h->iterations) h->iterations[k] = it;
      if (h && h->residual) h->residual[k] = g.last_rel;
      if (h && h->full_state) {
        g.gather_state(full.p);
        d2h(h->full_state + (size_t)(k + 1) * g.NSTATE, full.p, g.NSTATE, g.stream());
      }
    }
    if (np) {
      const size_t w = 2 + g.NT, S1 = n_steps + 1;
      std::vector<double> ph(S1 * np * w);
      SGW_CUDA(cudaMemcpyAsync(ph.data(), g.probe_hist.p, ph.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               g.stream()));
      SGW_CUDA(cudaStreamSynchronize(g.stream()));
      for (int p = 0; p < np; ++p)
        for (size_t k = 0; k < S1; ++k) {
          const double* o = &ph[(k * np + p) * w];
          if (h->probe_mean) h->probe_mean[p * S1 + k] = o[0];
          if (h->probe_std) h->probe_std[p * S1 + k] = o[1];
          if (h->probe_coeffs)
            for (int j = 0; j < g.NT; ++j) h->probe_coeffs[(p * g.NT + j) * S1 + k] = o[2 + j];
        }
    }
  });
}

int sgw_stats(sgw_solver* s, double* o) {
  return guard([&] {
    GpuSolver& g = *s->g;
    o[0] = g.setup_s;
    o[1] = g.T.pcg_ms;
    o[2] = g.T.step_ms;
    o[3] = double(g.T.iterations);
    o[4] = double(g_launches.load());
    o[5] = double(g.T.steps);
    o[6] = g.T.rhs_ms;
    o[7] = g.T.rec_ms;
    o[8] = double(g.T.matvecs);
    o[9] = double(g.T.nn2s);
  });
}

int sgw_reset_stats(sgw_solver* s) {
  return guard([&] {
    s->g->T = Timers{};
    s->g->KP.reset();
    SGW_CUDA(cudaMemset(s->g->tphase_.p, 0, 8 * sizeof(double)));
  });
}

int sgw_kernel_profile(sgw_solver* s, int enable, double* out) {
  return guard([&] {
    GpuSolver& g = *s->g;
    g.KP.on = enable != 0;
    if (out) {
      const double bytes[K_NCLASS] = {g.bytes_S(), g.bytes_Q(), g.bytes_sweep(), g.bytes_sgop()};
      for (int c = 0; c < K_NCLASS; ++c) {
        out[3 * c] = g.KP.ms[c];
        out[3 * c + 1] = double(g.KP.count[c]);
        out[3 * c + 2] = bytes[c];
      }
      out[12] = g.bytes_iter();
      double tp[8] = {0};
      SGW_CUDA(cudaMemcpy(tp, g.tphase_.p, sizeof(tp), cudaMemcpyDeviceToHost));
      for (int i = 0; i < 8; ++i) out[13 + i] = tp[i] * 1e-6;  // ms per phase, persistent PCG
      out[21] = g.flops_sgop();
    }
  });
}

// reads n doubles (the sum is written only if it is NaN, which it never is)
__global__ void l2_flush_read_kernel(const double* __restrict__ p, long long n, double* sink) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc += __ldcg(p + i);
  if (acc != acc) *sink = acc;
}

int sgw_bench_kernel(sgw_solver* s, int which, int reps, double* out) {
  return guard([&] {
    GpuSolver& g = *s->g;
    if (reps < 1) throw Error(SGW_EINVAL, "reps must be >= 1");
    DBuf<double> x, y;
    const size_t len = which >= 2 ? g.NSTATE : (size_t)g.NG;
    x.alloc(len), y.alloc(len);
    std::vector<double> h(len);
    for (size_t i = 0; i < len; ++i) h[i] = std::sin(0.001 * double(i) + 0.3);
    SGW_CUDA(cudaMemcpy(x.p, h.data(), len * sizeof(double), cudaMemcpyHostToDevice));
    auto once = [&] {
      if (which == 0) g.schur_matvec(x.p, y.p);
      else if (which == 1) g.apply_nn2(x.p, y.p);
      else if (which == 2) g.apply_block(2, x.p, y.p);
      else throw Error(SGW_EINVAL, "bench_kernel: which must be 0 (matvec), 1 (nn2), 2 (sg-op)");
    };
    once();
    cudaEvent_t a, b;
    SGW_CUDA(cudaEventCreate(&a));
    SGW_CUDA(cudaEventCreate(&b));
    float total = 0;
    if (which >= 2) {
      // the SG operator's couplings (~110 MB at C2) are about the L2 size: flush
      // L2 before every timed launch so that each one streams from HBM.  The
      // flush READS a 512 MB buffer: L2 is left holding clean lines, so the
      // timed kernel does not share HBM with the write-back of a memset.
      DBuf<double> flush;
      DBuf<double> sink;
      flush.alloc(size_t(64) << 20), sink.alloc(1);
      SGW_CUDA(cudaMemsetAsync(flush.p, 0, flush.n * sizeof(double), g.stream()));
      for (int r = 0; r < reps; ++r) {
        l2_flush_read_kernel<<<4 * 148, 512, 0, g.stream()>>>(flush.p, (long long)flush.n, sink.p);
        SGW_CUDA(cudaEventRecord(a, g.stream()));
        once();
        SGW_CUDA(cudaEventRecord(b, g.stream()));
        SGW_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        total += ms;
      }
    } else {
      SGW_CUDA(cudaEventRecord(a, g.stream()));
      for (int r = 0; r < reps; ++r) once();
      SGW_CUDA(cudaEventRecord(b, g.stream()));
      SGW_CUDA(cudaEventSynchronize(b));
      cudaEventElapsedTime(&total, a, b);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    g.KP.collect();
    out[0] = total / reps;
  });
}


int sgw_schur_from_locals(long long n_global, long long n_corner, int n_locals, const sgw_local_schur* locals,
                          sgw_schur** out) {
  return guard([&] {
    *out = nullptr;
    if (n_locals < 0 || (n_locals > 0 && !locals)) throw Error(SGW_EINVAL, "schur_from_locals: no locals");
    std::vector<GenericSchur::LocalInput> in(n_locals);
    for (int s = 0; s < n_locals; ++s) {
      const sgw_local_schur& l = locals[s];
      in[s].n = l.n, in[s].nr = l.nr, in[s].nc = l.nc;
      in[s].S = l.S, in[s].gmap = l.gmap, in[s].weights = l.weights;
      in[s].r_idx = l.r_idx, in[s].c_idx = l.c_idx, in[s].corner_gmap = l.corner_gmap;
    }
    auto h = std::make_unique<sgw_schur>();
    h->g = std::make_unique<GenericSchur>(n_global, n_corner, in);
    *out = h.release();
  });
}

void sgw_schur_free(sgw_schur* h) { delete h; }


int sgw_gschur_matvec(sgw_schur* h, const double* x, double* y) {
  return gschur_apply(h, x, y, [](GenericSchur& g, const double* a, double* b) { g.matvec(a, b); });
}

int sgw_gschur_apply_nn2(sgw_schur* h, const double* r, double* z) {
  return gschur_apply(h, r, z, [](GenericSchur& g, const double* a, double* b) { g.apply_nn2(a, b); });
}

int sgw_gschur_coarse_operator(sgw_schur* h, double* F) {
  return guard([&] {
    const auto& f = h->g->coarse_operator();
    std::memcpy(F, f.data(), f.size() * sizeof(double));
  });
}

int sgw_gschur_pcg(sgw_schur* h, const double* b, double tol, int max_iter, double* x, int* iterations,
                   int* converged, double* hist, int hist_cap, int* hist_len) {
  return guard([&] {
    GenericSchur& g = *h->g;
    const long long n = g.n_global();
    DBuf<double> db, dx;
    db.alloc(std::max<long long>(1, n)), dx.alloc(std::max<long long>(1, n));
    SGW_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, g.stream()));
    bool conv = false;
    std::vector<double> hh;
    const int it = pcg_generic(
        g.blas(), g.stream(), n, [&](const double* a, double* c) { g.matvec(a, c); },
        [&](const double* a, double* c) { g.apply_nn2(a, c); }, db.p, dx.p, tol, max_iter, &conv, &hh);
    SGW_CUDA(cudaMemcpy(x, dx.p, n * 8, cudaMemcpyDeviceToHost));
    report_out(it, conv, hh, iterations, converged, hist, hist_cap, hist_len);
  });
}

int sgw_pcg_ops(long long n, sgw_host_op op, void* op_ctx, sgw_host_op precond, void* precond_ctx, const double* b,
                double tol, int max_iter, double* x, int* iterations, int* converged, double* hist, int hist_cap,
                int* hist_len) {
  return guard([&] {
    if (!op || n < 0) throw Error(SGW_EINVAL, "pcg: no operator");
    cudaStream_t st;
    cublasHandle_t blas;
    SGW_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) throw Error(SGW_ECUDA, "cublasCreate failed");
    cublasSetStream(blas, st);
    struct Cleanup {
      cudaStream_t s;
      cublasHandle_t b;
      ~Cleanup() {
        cublasDestroy(b);
        cudaStreamDestroy(s);
      }
    } cleanup{st, blas};
    std::vector<double> hx(std::max<long long>(1, n)), hy(std::max<long long>(1, n));
    auto host_op = [&](sgw_host_op f, void* ctx) {
      return [&, f, ctx](const double* a, double* c) {
        SGW_CUDA(cudaMemcpyAsync(hx.data(), a, n * 8, cudaMemcpyDeviceToHost, st));
        SGW_CUDA(cudaStreamSynchronize(st));
        if (f) f(ctx, n, hx.data(), hy.data());
        else std::memcpy(hy.data(), hx.data(), n * 8);
        SGW_CUDA(cudaMemcpyAsync(c, hy.data(), n * 8, cudaMemcpyHostToDevice, st));
        SGW_CUDA(cudaStreamSynchronize(st));
      };
    };
    DBuf<double> db, dx;
    db.alloc(std::max<long long>(1, n)), dx.alloc(std::max<long long>(1, n));
    SGW_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, st));
    bool conv = false;
    std::vector<double> hh;
    const int it = pcg_generic(blas, st, n, host_op(op, op_ctx), host_op(precond, precond_ctx), db.p, dx.p, tol,
                               max_iter, &conv, &hh);
    SGW_CUDA(cudaMemcpy(x, dx.p, n * 8, cudaMemcpyDeviceToHost));
    report_out(it, conv, hh, iterations, converged, hist, hist_cap, hist_len);
  });
}

int sgw_kle_spectrum(double sigma, double bx, double by, int n_vars, double* out) {
  return guard([&] {
    const auto l = kle_spectrum(sigma, bx, by, n_vars);
    std::memcpy(out, l.data(), l.size() * sizeof(double));
  });
}

int sgw_pce_indices(int n_vars, int order, int* out, long long cap, int* n_terms) {
  return guard([&] {
    const auto ix = pce_indices(n_vars, order);
    *n_terms = int(ix.size());
    if (out) {
      if ((long long)ix.size() * n_vars > cap) throw Error(SGW_EINVAL, "index buffer too small");
      for (size_t k = 0; k < ix.size(); ++k) std::memcpy(out + k * n_vars, ix[k].data(), n_vars * sizeof(int));
    }
  });
}

int sgw_lognormal_coeff(int nx, int ny, double sigma, double bx, double by, double g0, int n_vars, int p_in,
                        double* out, long long cap, int* n_in) {
  return guard([&] {
    const auto c = lognormal_coeff(nx, ny, sigma, bx, by, g0, n_vars, p_in);
    *n_in = int(c.size());
    if (out) {
      const size_t nn = (size_t)(nx + 1) * (ny + 1);
      if ((long long)(c.size() * nn) > cap) throw Error(SGW_EINVAL, "coefficient buffer too small");
      for (size_t i = 0; i < c.size(); ++i) std::memcpy(out + i * nn, c[i].data(), nn * sizeof(double));
    }
  });
}

int sgw_triple_products(int n_vars, int p_in, int p_out, int* n_in, int* n_out, int* n_entries, int* ei, int* ej,
                        int* ek, double* ev, long long cap) {
  return guard([&] {
    const TensorHost t = triple_products(n_vars, p_in, p_out);
    *n_in = t.n_in;
    *n_out = t.n_out;
    *n_entries = int(t.v.size());
    if (ei) {
      if ((long long)t.v.size() > cap) throw Error(SGW_EINVAL, "tensor buffer too small");
      for (size_t e = 0; e < t.v.size(); ++e) ei[e] = t.i[e], ej[e] = t.j[e], ek[e] = t.k[e], ev[e] = t.v[e];
    }
  });
}

int sgw_nearest_node(int nx, int ny, double x, double y) { return nearest_node(nx, ny, x, y); }

int sgw_shard_plan(int nx, int ny, int px, int py, int world, int rank, long long* info, int* sub_owner,
                   int* iface_gpos, int* peers, int* peer_off, int* peer_idx) {
  return guard([&] {
    if (!info) throw Error(SGW_EINVAL, "null argument");
    const Geometry g = build_geometry(nx, ny, px, py, rank, world);
    const Halo& h = g.halo;
    info[0] = g.rx, info[1] = g.ry, info[2] = g.ns, info[3] = g.n_iface, info[4] = (long long)h.peers.size();
    info[5] = (long long)h.idx.size(), info[6] = g.n_iface_global;
    if (sub_owner)
      for (int s2 = 0; s2 < g.ns_total; ++s2) sub_owner[s2] = g.rank_of_sub(s2);
    if (iface_gpos) std::memcpy(iface_gpos, g.iface_gpos.data(), g.iface_gpos.size() * sizeof(int));
    if (peers) std::memcpy(peers, h.peers.data(), h.peers.size() * sizeof(int));
    if (peer_off) std::memcpy(peer_off, h.peer_off.data(), h.peer_off.size() * sizeof(int));
    if (peer_idx) std::memcpy(peer_idx, h.idx.data(), h.idx.size() * sizeof(int));
  });
}

int sgw_nccl_unique_id(void* out128) {
  return guard([&] {
    if (!out128) throw Error(SGW_EINVAL, "null argument");
    nccl_unique_id(out128);
  });
}

}  // extern "C"
