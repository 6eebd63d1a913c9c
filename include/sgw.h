/*
 * sgw.h — C ABI of the B200-native SG-PCG / NN2 solver (libsgw_b200.so).
 *
 * Drop-in boundary for the reference sgwave hot path: the per-Newmark-step
 * interface-Schur PCG solve of the coupled (P+1) x N stochastic-Galerkin
 * system, preconditioned by the probabilistic two-level Neumann-Neumann
 * (NN2) domain decomposition.  Every entry point takes plain pointers and
 * sizes (host memory unless the name says _dev), returns an sgw_status and
 * never retains caller pointers past the call.  Error text for the last
 * failing call on the calling thread: sgw_last_error().
 *
 * Reference interfaces replaced (paths relative to the reference proj/):
 *   sgw_create          SgSolver::SgSolver            include/sgwave/sg.hpp:45-47, src/sg.cpp:128-176
 *                       (+ assemble_subdomains src/sg.cpp:178-250, SchurSystem::finalize src/dd.cpp:98-140)
 *   sgw_run             SgSolver::run                 include/sgwave/sg.hpp:49-50, src/sg.cpp:358-423
 *   sgw_init_state /    SgSolver::run's time loop split into resident steps
 *   sgw_advance         (step_rhs_and_solve src/sg.cpp:295-356 + newmark_update src/newmark.cpp:39-49)
 *   sgw_apply_block     SgSolver::apply_block_{mass,stiffness,transient}  sg.hpp:58-60, src/sg.cpp:425-447
 *   sgw_schur_matvec    SchurSystem::matvec           include/sgwave/dd.hpp:85, src/dd.cpp:142-157
 *   sgw_apply_nn2       SchurSystem::apply_nn2        include/sgwave/dd.hpp:88, src/dd.cpp:199-253
 *   sgw_apply_precond   make_preconditioner / apply_{lumped,nn1,nn2}  dd.hpp:86-88,102, src/dd.cpp:159-253
 *   sgw_pcg             pcg(matvec, apply_nn2, ...)   include/sgwave/pcg.hpp:20-21, src/pcg.cpp:7-50
 *   sgw_coarse_operator SchurSystem::coarse_operator  include/sgwave/dd.hpp:90
 *   sgw_schur_from_locals / sgw_gschur_*  SchurSystem built from LocalSchur data  dd.hpp:50-96
 *   sgw_pcg_ops         pcg(LinearOp, LinearOp, ...)  include/sgwave/pcg.hpp:15-21, src/pcg.cpp:7-50
 *   sgw_lognormal_coeff lognormal_pce(kle_exponential(...))  src/lognormal.cpp:8-40, src/kle.cpp:80-133
 *   sgw_triple_products triple_products               src/pce.cpp:96-122 (order_in <= order_out guard lifted)
 *   sgw_nearest_node    nearest_node                  src/mesh.cpp:83-96
 *   sgw_kle_spectrum    kle_spectrum_csv's lambdas    src/kle.cpp:161-167
 *   sgw_pce_indices     PceBasis::indices_csv's rows  src/pce.cpp:84-94
 *
 * Error classes (reference exception -> status):
 *   std::invalid_argument (sg.cpp:143-145, :382)            -> SGW_EINVAL
 *   std::runtime_error factorization (sg.cpp:151,:170,:221; dd.cpp:72-74) -> SGW_EFACTOR
 *   std::runtime_error non-convergence (sg.cpp:413-416)      -> SGW_ENOCONV
 *   CUDA / cuBLAS / cuSOLVER failures                        -> SGW_ECUDA
 *   NCCL failures (multi-GPU)                                -> SGW_ENCCL
 */
#ifndef SGW_H_
#define SGW_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sgw_status {
  SGW_OK = 0,
  SGW_EINVAL = 1,
  SGW_EFACTOR = 2,
  SGW_ENOCONV = 3,
  SGW_ECUDA = 4,
  SGW_ENCCL = 5,
  SGW_ENOMEM = 6
} sgw_status;

typedef struct sgw_solver sgw_solver;

/* SgSolver constructor arguments.  The mesh is build_unit_square_mesh(nx, ny)
 * (src/mesh.cpp:15-58) and the partition partition_structured(mesh, px, py)
 * (src/partition.cpp:48-133), floor-division cell ownership: px need not
 * divide nx (ragged blocks of two widths are supported).                   */
typedef struct sgw_problem {
  int nx, ny, px, py;
  int n_input;          /* CoefficientField terms                              */
  const double* coeff;  /* n_input x (nx+1)(ny+1) nodal values, term-major     */
  int n_output;         /* TripleTensor::n_output  (P+1)                       */
  int n_entries;        /* TripleTensor entries with j <= k (pce.hpp:24-40)    */
  const int* ent_i;
  const int* ent_j;
  const int* ent_k;
  const double* ent_v;
  double density, alpha0, alpha1;
  double gamma, zeta, dt; /* NewmarkParams (newmark.hpp:11-19)                 */
  double tol;             /* SgOptions::tol (sg.hpp:16)                         */
  int max_iter;           /* SgOptions::max_iter                               */
  int device;             /* CUDA device ordinal                                */
  /* Multi-GPU sharding (one process per GPU); world_size 1 = single GPU.
   * The ranks form an rx x ry grid (sgw_shard_plan) and each owns a 2D block
   * of subdomains and the interface nodes they touch; interface sums are
   * completed by point-to-point halo exchanges (ncclSend/ncclRecv) with the
   * neighbouring ranks, the coarse vector and the CG scalars by
   * ncclAllReduce.  Every entry point is collective: all ranks call it with
   * the same arguments.  Results (state, probes, PCG output) are identical on
   * all ranks; interface vectors at this boundary are always global.
   * nccl_id: 128-byte ncclUniqueId from sgw_nccl_unique_id on rank 0,
   * broadcast by the caller (e.g. torch.distributed).  A non-NULL id with
   * world_size 1 runs the sharded code path on a 1-rank communicator.      */
  int rank, world_size;
  const void* nccl_id;
  /* PrecondKind (dd.hpp:98) of the PCG: 0 nn2 (the SG path, sg.cpp:330),
   * 1 nn1 (dd.cpp:178-195), 2 lumped (dd.cpp:159-176, gg_action = the
   * flattened A_GG block as DetSolver's K~_GG, det_loop.cpp:165-167).
   * DetSolver::set_preconditioner / SolveOptions::precond (det_loop.hpp:14). */
  int precond;
  /* Reduced-memory mode: 1 = the local Schur complements S_s
   * are not stored; every S product applies A_GG - A_GI A_II^-1 A_IG per
   * subdomain through the local stencils and one batched interior solve
   * (sg.cpp:227-245 formed on the fly).  NN2 keeps its explicit S_rr^-1,
   * Psi and F_cc^-1.  Saves the S tiles (1.3 GB at C2, 18 GB at C3) at the
   * cost of one interior sweep per PCG iteration.                          */
  int implicit_schur;
} sgw_problem;

/* ForceFn (det_loop.hpp:32): kind 0 none; 1 Ricker wavelet
 *   amp * (1 - 2 pi^2 f0^2 (t - t0)^2) exp(-pi^2 f0^2 (t - t0)^2) at mesh node `node`;
 * 2 nodal table, (n_steps + 1) x n_nodes rows for t_0 .. t_N, read straight
 *   from the caller's buffer during sgw_run (it must stay valid until sgw_run
 *   returns; the solver drops it afterwards).                                */
typedef struct sgw_force {
  int kind;
  int node;
  double f0, t0, amp;
  const double* table;
} sgw_force;

/* SgHistory (sg.hpp:23-31).  Caller-owned output buffers; NULL = not wanted. */
typedef struct sgw_history {
  int* iterations;       /* n_steps                                   */
  double* residual;      /* n_steps: final true residual ||b-Ax||/||b|| */
  int n_probes;
  const int* probe_nodes;/* mesh node ids                               */
  double* probe_mean;    /* n_probes x (n_steps + 1)                    */
  double* probe_std;     /* n_probes x (n_steps + 1)                    */
  double* full_state;    /* (n_steps + 1) x (P+1) n_dofs, term-major    */
  double* probe_coeffs;  /* n_probes x (P+1) x (n_steps + 1): every chaos
                            coefficient at the probes (SgHistory::probe_coeffs) */
} sgw_history;

const char* sgw_last_error(void);
int sgw_version(void);

int sgw_create(const sgw_problem* problem, sgw_solver** out);
int sgw_destroy(sgw_solver* s);

/* sizes: [0] n_dofs  [1] n_terms  [2] n_iface  [3] n_corner  [4] n_global (flat)
 *        [5] n_sub   [6] uses_direct (always 0 on the GPU path)  [7] device bytes */
int sgw_sizes(sgw_solver* s, long long* sizes);

/* Launch all work on this cudaStream_t (NULL = library-owned stream). */
int sgw_set_stream(sgw_solver* s, void* cuda_stream);

/* op: 0 mass, 1 stiffness, 2 transient.  x, y: (P+1) n_dofs, term-major.   */
int sgw_apply_block(sgw_solver* s, int op, const double* x, double* y);
int sgw_schur_matvec(sgw_solver* s, const double* x, double* y);
int sgw_apply_nn2(sgw_solver* s, const double* r, double* z);
/* make_preconditioner(schur, kind)(r) (dd.cpp): kind 0 nn2, 1 nn1, 2 lumped;
 * nn1 / lumped need problem->precond == kind (SGW_EINVAL otherwise).       */
int sgw_apply_precond(sgw_solver* s, int kind, const double* r, double* z);
/* PCG on S u = rhs with NN2 (src/pcg.cpp:7-50).  history: >= max_iter + 2. */
int sgw_pcg(sgw_solver* s, const double* rhs, double* x, int* iterations, int* converged,
            double* residual_history, int history_cap);
/* Verification hook (test_dd.cpp:77-96 at full size): dense copy of global
 * subdomain `sub`'s local operator, column-major: which 0 = S_s (a x a),
 * 1 = S_rr^-1 (r x r), 2 = Psi_s = S_rr^-1 S_rc (r x c).  dims (optional) =
 * {a, r, c}; gmap (optional, a entries) = make_flat_maps' gmap (dd.cpp:78-96).
 * out = gmap = NULL: sizes only.  The subdomain must be owned by this rank. */
int sgw_local_block(sgw_solver* s, int sub, int which, double* out, long long* gmap, long long* dims);
/* F_cc (n_corner flat)^2, column-major. */
int sgw_coarse_operator(sgw_solver* s, double* out);

int sgw_run(sgw_solver* s, const double* u0_nodal, const double* v0_nodal, int n_steps,
            const sgw_force* force, sgw_history* history);

/* Device-resident stepping (for benchmarks): set the initial state and the
 * forcing, then advance n steps without host round trips of the state.
 * A step whose interface solve does not converge returns SGW_ENOCONV and
 * leaves the state, the time and the step index where they were
 * (sg.cpp:412-416), also when the following step's right-hand side was
 * already queued behind it.                                               */
int sgw_init_state(sgw_solver* s, const double* u0_nodal, const double* v0_nodal,
                   const sgw_force* force);
int sgw_advance(sgw_solver* s, int n_steps, int* iterations);
int sgw_get_state(sgw_solver* s, double* u_flat);

/* stats: [0] setup s  [1] pcg ms (device events, last advance/run)
 *        [2] step ms  [3] PCG iterations  [4] kernel launches  [5] steps
 *        [6] rhs ms   [7] recovery ms     [8] matvec calls    [9] nn2 calls */
int sgw_stats(sgw_solver* s, double* out);
int sgw_reset_stats(sgw_solver* s);

/* Per-kernel-class device timing (CUDA events around each launch on the
 * solver stream).  enable: 1 on / 0 off.  out (optional, 12 doubles): for
 * classes {S tile-SYMV, Q tile-SYMV, interior sweep, SG-operator apply}:
 * [total ms, launches, algorithmic bytes per launch]; out[12] = algorithmic
 * bytes of one PCG iteration (SURVEY 8d B_iter); out[13..20] = critical-path
 * ms of the 8 phases of the persistent PCG kernel; out[21] = algorithmic
 * flops of one SG-operator apply.  out needs 22 doubles.                   */
int sgw_kernel_profile(sgw_solver* s, int enable, double* out);
/* Average device ms of `reps` back-to-back calls of one operation:
 * which 0 = Schur matvec, 1 = NN2 apply, 2 = global transient SG operator.  */
int sgw_bench_kernel(sgw_solver* s, int which, int reps, double* out_ms);

/* Interface systems from caller-built local Schur data (the reference's
 * LocalSchur fields, include/sgwave/dd.hpp:50-62, as test_dd.cpp:123-151
 * builds one by hand): SchurSystem{n_global, n_corner, locals}.finalize(),
 * matvec, apply_nn2, coarse_operator and pcg(matvec, apply_nn2, ...) on the
 * GPU (src/dd.cpp:98-157, :199-253; src/pcg.cpp:7-50).  S is n x n
 * column-major; every array is copied.                                     */
typedef struct sgw_local_schur {
  int n;                         /* flat local interface size */
  const double* S;               /* n x n local Schur complement */
  const long long* gmap;         /* n: local -> global flat interface index */
  const double* weights;         /* n: partition-of-unity weights D_s */
  int nr;                        /* remaining (non-corner) local indices */
  const int* r_idx;
  int nc;                        /* corner local indices */
  const int* c_idx;
  const long long* corner_gmap;  /* nc: corner -> global corner index */
} sgw_local_schur;
typedef struct sgw_schur sgw_schur;
int sgw_schur_from_locals(long long n_global, long long n_corner, int n_locals, const sgw_local_schur* locals,
                          sgw_schur** out);
void sgw_schur_free(sgw_schur* h);
int sgw_gschur_matvec(sgw_schur* h, const double* x, double* y);
int sgw_gschur_apply_nn2(sgw_schur* h, const double* r, double* z);
int sgw_gschur_coarse_operator(sgw_schur* h, double* F);  /* n_corner^2, column-major */
/* pcg(matvec, apply_nn2, b, tol, max_iter) on this system (x0 = 0). */
int sgw_gschur_pcg(sgw_schur* h, const double* b, double tol, int max_iter, double* x, int* iterations,
                   int* converged, double* hist, int hist_cap, int* hist_len);

/* pcg (include/sgwave/pcg.hpp:15-21, src/pcg.cpp:7-50) over caller-supplied
 * operators, the reference's LinearOp: op(ctx, n, x, y) writes y = A x for
 * host vectors of length n (precond: z = M^-1 r; NULL = identity).  The CG
 * recurrence (vectors, dots, axpys) runs on the GPU; each operator call
 * copies its input to the host and its output back.  Report as sgw_pcg.   */
typedef void (*sgw_host_op)(void* ctx, long long n, const double* x, double* y);
int sgw_pcg_ops(long long n, sgw_host_op op, void* op_ctx, sgw_host_op precond, void* precond_ctx, const double* b,
                double tol, int max_iter, double* x, int* iterations, int* converged, double* hist, int hist_cap,
                int* hist_len);

/* Input builders (host). */
int sgw_lognormal_coeff(int nx, int ny, double sigma, double bx, double by, double g0,
                        int n_vars, int p_in, double* out, long long out_cap, int* n_in);
int sgw_triple_products(int n_vars, int p_in, int p_out, int* n_in, int* n_out, int* n_entries,
                        int* ei, int* ej, int* ek, double* ev, long long cap);
int sgw_nearest_node(int nx, int ny, double x, double y);
/* kle_spectrum.csv / pce_indices.csv inputs (src/kle.cpp:161-167,
 * src/pce.cpp:84-94): the n_vars sorted KLE eigenvalues of the separable
 * exponential covariance times sigma^2 (out: n_vars doubles); the PCE multi-indices of
 * total order <= order in basis order (out: n_terms x n_vars, row-major; out
 * may be NULL to query n_terms).                                             */
int sgw_kle_spectrum(double sigma, double bx, double by, int n_vars, double* out);
int sgw_pce_indices(int n_vars, int order, int* out, long long out_cap, int* n_terms);

/* Sharding plan (host only, no GPU needed): the rx x ry rank grid and rank
 * `rank`'s halo.  info[7] = {rx, ry, owned subdomains, local interface nodes,
 * peers, shared entries (sum over peers), global interface nodes}.  Optional
 * outputs: sub_owner[px py] (rank of every subdomain), iface_gpos[local
 * nodes] (global interface position of each local node, ascending), peers[],
 * peer_off[peers + 1] and peer_idx[shared entries] (per peer, the shared
 * local nodes in ascending global position).  Call with NULLs to size.       */
int sgw_shard_plan(int nx, int ny, int px, int py, int world, int rank, long long* info, int* sub_owner,
                   int* iface_gpos, int* peers, int* peer_off, int* peer_idx);
/* NCCL unique id for multi-GPU runs (128 bytes), generated on rank 0. */
int sgw_nccl_unique_id(void* out128);

/* In-process sharding on ONE device (tests): world_size solvers, each driven
 * by its own host thread, exchange through a host-synchronised group
 * instead of NCCL.  Same ownership and results as the NCCL path.           */
int sgw_local_group_new(int world_size, void** group);
/* One rank of a world_size-rank decomposition constructed alone on one device
 * (no peers: every exchange delivers zeros, the coarse matrix holds only this
 * rank's subdomains).  For per-rank memory and shard-kernel timing of
 * configurations that need several GPUs (C4); results are not physical.     */
int sgw_create_solo(const sgw_problem* problem, int world_size, int rank, sgw_solver** out);
int sgw_local_group_free(void* group);
/* a failed rank's thread releases the others: their pending and later
 * collectives fail with SGW_ENCCL instead of waiting forever.            */
int sgw_local_group_abort(void* group);
int sgw_create_local_group(const sgw_problem* problem, int world_size, int rank, void* group,
                           sgw_solver** out);

#ifdef __cplusplus
}
#endif
#endif /* SGW_H_ */
