// Host side of the B200 implicit MPM Newton step: device state, the Newton
// controller (a line-for-line behavioural restatement of
// /root/reference/proj/include/impm/mpm_solver.hpp:93-407 over device
// kernels), the Krylov solve that replaces sparse_lu_solve
// (src/linear_solver.cpp:11-88), and the C ABI of include/impm_gpu.h.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/impm_gpu.h"
#include "impm_kernels.cuh"
#include "impm_comm.cuh"

using namespace impm_gpu;

namespace {

// kernel launches issued by this library (every <<<>>> is followed by ++g_launches)
std::atomic<long long> g_launches{0};

// ----------------------------------------------------------- errors -----
struct SimError : std::runtime_error {
  impm_status code;
  std::vector<double> history;
  SimError(impm_status c, const std::string& m, std::vector<double> h = {})
      : std::runtime_error(m), code(c), history(std::move(h)) {}
};

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw SimError(IMPM_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e_) +     \
                                        " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define CKL() CK(cudaGetLastError())

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  // a buffer that has to grow gets 1/8 headroom: the active set of a load
  // ramp grows a little every step, and a cudaFree + cudaMalloc of the 6 GB
  // matrix (an implicit device sync) each time costs milliseconds
  void ensure(size_t n) {
    if (n <= cap && p) return;
    const bool regrow = p != nullptr;
    if (p) CK(cudaFree(p));
    p = nullptr;
    size_t c = std::max<size_t>(n, 1);
    if (regrow) c += static_cast<size_t>(static_cast<double>(c) * buf_slack());
    CK(cudaMalloc(&p, c * sizeof(T)));
    cap = c;
  }
  static double buf_slack() {
    static const double f = std::getenv("IMPM_BUF_SLACK") ? std::atof(std::getenv("IMPM_BUF_SLACK")) : 0.125;
    return f;
  }
  T* get() const { return p; }
};

constexpr int kThreads = 256;
constexpr int kRedBlocks = 148 * 4;    // fixed partial count for deterministic reductions
constexpr int kSpmvBlocks = 148 * 8;   // SpMV grid: 4-warp CTAs, 8 resident per SM -> exactly one wave
constexpr int kSpmvMaxBlocks = 148 * 32;
inline unsigned blocks_for(int64_t n, int t = kThreads) { return static_cast<unsigned>(std::max<int64_t>(1, (n + t - 1) / t)); }

template <int V>
using IC = std::integral_constant<int, V>;

// ---------------------------------------------------------- profiling ---
enum KClass {
  kcSort = 0, kcMass, kcDof, kcResP, kcResN, kcTangent, kcAssemble, kcSpmv, kcKrylov, kcCommit, kcMgSetup, kcVcycle,
  kcGalerkin, kcMgPower, kcMgCoarsest, kcVcL0, kcVcL1, kcVcCoarse, kcCount
};
const char* kClassNames[kcCount] = {"support_sort", "node_mass", "dof_map", "residual_particles", "residual_nodes",
                                    "tangent",      "assemble",  "spmv",    "krylov_vector",      "commit",
                                    "mg_setup",     "vcycle",    "galerkin", "mg_power",           "mg_coarsest",
                                    "vcycle_level0", "vcycle_level1", "vcycle_coarse"};

struct Prof {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  double ms[kcCount] = {};
  int64_t launches[kcCount] = {};
  size_t used = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  struct Scope {
    Prof* p;
    int cls;
    cudaEvent_t b{}, e{};
    Scope(Prof* pr, int c) : p(pr), cls(c) {
      if (p->on) {
        b = p->ev();
        e = p->ev();
        CK(cudaEventRecord(b, p->s));
      }
    }
    ~Scope() {
      if (p->on) {
        cudaEventRecord(e, p->s);
        p->pending.push_back({cls, {b, e}});
      }
    }
  };
  void flush() {  // caller has synchronized the stream
    for (auto& q : pending) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, q.second.first, q.second.second) == cudaSuccess) {
        ms[q.first] += t;
        launches[q.first] += 1;
      }
    }
    pending.clear();
    used = 0;
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// ---------------------------------------------------------- multigrid ---
}  // namespace

// device CSR linear algebra (the sparse_lu_solve seam), also the direct path of
// the Newton solve on small systems
#include "impm_csr.cuh"

namespace {

struct MgLevel {
  GridC g{};
  int n_act = 0;
  int64_t row_len = 0;
  // owned storage (coarse levels; level 0 views the fine Jacobian)
  DBuf<int> act_flag_b, act_scan_b, act_idx_b, act_list_b, row_nzb_b;
  DBuf<uint8_t> freem_b, row_slots_b;
  DBuf<double> vals_b, dinv_b;
  DBuf<float> vals32_b;          // fp32 copy for the smoother / residual SpMVs
  DBuf<__half> vals16_b;         // fp16 row-scaled copy (big coarse levels)
  DBuf<float> rscale_b;
  DBuf<double> xa, xb, r, bvec;  // level vectors (grid layout)
  DBuf<float> x4a, x4b;          // fp32 twins of xa / xb, 4 floats per node (fp32 SpMV gathers)
  // views
  const int* act_idx = nullptr;
  const int* act_list = nullptr;
  const int* row_nzb = nullptr;
  const uint8_t* freem = nullptr;
  const uint8_t* row_slots = nullptr;
  const double* vals = nullptr;
  const float* vals32 = nullptr;
  int64_t row_len32 = 0;
  const __half* vals16 = nullptr;  // fine level only: fp16 smoother copy + row scales
  const float* rscale = nullptr;
  int64_t row_len16 = 0;
  const double* dinv = nullptr;
  double* x = nullptr;  // current iterate (ping-pong between xa / xb)
  double* t = nullptr;
  float* twin(const double* v) { return v == xa.p ? x4a.p : (v == xb.p ? x4b.p : nullptr); }
  double omega = 0.5;
};

// ------------------------------------------------------------ the sim ---
struct Sim {
  // configuration
  int D = 2, F = 2, shape = 1;
  GridC g{};
  impm_material mat{};
  impm_options opt{};
  double gravity[3] = {0, 0, 0};
  int device = 0;
  cudaStream_t own_stream = nullptr, s = nullptr;

  // particles
  int P = 0;
  int64_t cap = 0;
  int ND = 0;
  DBuf<double> pd, pd_tmp, xs, bext, Pst, Atan;
  DBuf<double> io_staging;  // AoS staging of particle upload / download
  DBuf<int> io_inv;         // original -> sorted slot (chunked download)
  // particle I/O in chunks: the host<->device copies run on io_stream and
  // overlap the layout kernels on s (IMPM_IO_CHUNKS=1: one copy, one kernel)
  static constexpr int kIoMaxChunks = 16;
  cudaStream_t io_stream = nullptr;
  cudaEvent_t io_ev[kIoMaxChunks + 1] = {};
  int io_chunks = std::getenv("IMPM_IO_CHUNKS") ? std::max(1, std::min(kIoMaxChunks, std::atoi(std::getenv("IMPM_IO_CHUNKS")))) : 8;
  DBuf<int> orig, orig_tmp, key, sup, rank, perm, bin_count, bin_start;
  // grid / dofs
  DBuf<uint8_t> fixed, freem;
  DBuf<int> act_flag, act_scan, act_idx, act_list, free_flag, free_scan, dof_of, node_of, field_of;
  DBuf<int> scan_sums_i, brick_flag, brick_scan;
  DBuf<int64_t> scan_sums_l, rowlen, rowptr;
  DBuf<double> mass;
  int n_dofs = 0, n_act = 0;
  // vectors (grid layout [N][F])
  DBuf<double> u, r, delta, utry, rtry, prev, tmp1, tmp2;
  DBuf<double> kx, kr, kz, kp, kq, kv, ks, kt, khat;
  // matrix
  DBuf<double> vals, dinv;
  DBuf<uint8_t> row_slots, bflag;
  DBuf<int> row_nzb;
  DBuf<unsigned> row_mask;
  DBuf<unsigned long long> nzb_total;
  unsigned long long h_nzb_total = 0;
  int64_t row_len = 0;
  bool matrix_valid = false;
  // multigrid hierarchy (rebuilt with every Jacobian)
  std::vector<std::unique_ptr<MgLevel>> mg;
  DBuf<double> mg_dense, mg_lam, mg_T;
  std::vector<double> mg_lam_host;
  int mg_power_step = -1;
  DBuf<unsigned long long> mg_nzb;
  int mg_dense_n = 0;
  unsigned long long mg_stored_blocks = 0;
  // reductions / status
  DBuf<double> partials, sums, sc;
  DBuf<DevStatus> st;
  DBuf<int> dflag;
  DevStatus* h_st = nullptr;  // pinned mirror
  double* h_sc = nullptr;

  // coupled u-p mode (CoupledSim, porous.hpp:48-125)
  bool coupled = false;
  PoroC pc{};
  double up_dt = 0.0, up_time = 0.0, up_rscale = 0.0;
  DBuf<double> uty;  // accumulated vertical displacement per particle (sorted order)

  int spmv_blocks = kSpmvBlocks;
  int mg_blocks = kSpmvBlocks;  // grid of the level sweeps without dot partials
  // the MG preconditioner streams fp32 copies of its level matrices (the
  // outer Krylov SpMV stays fp64, so the solve tolerance is unaffected)
  bool mg_f32 = true;
  DBuf<float> vals32;
  DBuf<__half> vals16;  // fp16 smoother copy of the fine J (row-scaled)
  DBuf<float> rscale16;
  // vals16 already holds the current J (written by the fused transpose pass)
  bool f16_ready = false;
  bool mirror_f16 = !(std::getenv("IMPM_MIRROR_F16") && std::atoi(std::getenv("IMPM_MIRROR_F16")) == 0);
  // coarse levels (Galerkin products, dense coarsest inverse) are kept for
  // the later Newton iterations of a load step: the row structure is fixed
  // within a step and J moves little, while the fine level always smooths
  // with the current J
  bool mg_reuse = true;
  int mg_setup_step = -1;
  // relative Krylov tolerance of the current solve (see newton_attempt)
  double cur_rtol = 1e-12;
  // |r1| / r0 of the last converged load step (first-iteration forcing term)
  double newton_ratio1 = -1.0;
  double newton_eta_factor = 0.01;
  int mg_smooth_env = 0;
  // 3D tangent: one dual direction per pass (160 registers, 9 passes) beats
  // three per pass (255 registers, 12% occupancy): 13.7 -> 10.3 ms per step
  bool tangent_k1 = true;
  // rebuild the coarse MG levels every mg_refresh load steps (A/B experiments)
  // (default 3; a solve on stale levels that fails or overruns 4x the last
  // iteration count is retried once on a freshly built hierarchy)
  // (cfg 4 at omega safety 1.0, Newton it/s: driver window 3: 13.12, 5: 13.00, 6: 13.35, 8: 12.94;
  // default window 3: 14.08, 6: 14.86; the capped stale-level solve keeps the Krylov counts)
  int mg_refresh = std::getenv("IMPM_MG_REFRESH") ? std::atoi(std::getenv("IMPM_MG_REFRESH")) : 6;
  // re-estimate the smoother's lambda_max every mg_power_every load steps (A/B experiments)
  int mg_power_every = std::getenv("IMPM_MG_POWER_EVERY") ? std::max(1, std::atoi(std::getenv("IMPM_MG_POWER_EVERY"))) : 5;
  // safety factor on the power estimate in omega = 4 / (3 s lambda): cfg 4 driver window,
  // Newton it/s (Krylov it): s = 1.2 12.05 (719), 1.1 12.33 (686), 1.0 12.69 (656),
  // 0.95 12.57 (670), 0.9 11.42 (stale-level retries), 0.8 3.37 (smoother diverges)
  double mg_omega_safety = std::getenv("IMPM_MG_OMEGA_SAFETY") ? std::atof(std::getenv("IMPM_MG_OMEGA_SAFETY")) : 1.0;
  double mg_omega_safety_coarse =
      std::getenv("IMPM_MG_OMEGA_SAFETY_COARSE") ? std::atof(std::getenv("IMPM_MG_OMEGA_SAFETY_COARSE")) : 0.0;
  // smoothing sweeps on the levels below the fine one (0: as the fine level; A/B experiments)
  int mg_nu_coarse = std::getenv("IMPM_MG_NU_COARSE") ? std::atoi(std::getenv("IMPM_MG_NU_COARSE")) : 0;
  double exact_rtol = 1e-13;         // Krylov target of an exact-equivalent Newton step
  int exact_newton_env = -1;         // IMPM_EXACT_NEWTON: -1 = by material
  bool exact_newton = false;         // set per material at create / set_material
  bool mg_cross_ok = false;  // set by cg_mg_solve around its capped solve on stale levels
  // assembly flush: per-lane RED.ADD.F64 (default) or the transposed plain RMW
  // (IMPM_ASM_RMW=1: 40 vs 34 ms per cfg 4 Jacobian);
  // symmetric mirroring for symmetric J (IMPM_ASM_SYM=0: full)
  // 3D neo-Hookean tangent in closed form (IMPM_TANGENT_DUAL=1: dual numbers)
  bool tangent_analytic = !(std::getenv("IMPM_TANGENT_DUAL") && std::atoi(std::getenv("IMPM_TANGENT_DUAL")) != 0);
  bool asm_rmw = std::getenv("IMPM_ASM_RMW") && std::atoi(std::getenv("IMPM_ASM_RMW")) != 0;
  bool asm_sym = !(std::getenv("IMPM_ASM_SYM") && std::atoi(std::getenv("IMPM_ASM_SYM")) == 0);
  // 3D neo-Hookean: factored tangent + pair-per-thread assembly (IMPM_ASM_NHF=0: dP/dG + k_assemble_bins_staged)
  bool asm_nhf = !(std::getenv("IMPM_ASM_NHF") && std::atoi(std::getenv("IMPM_ASM_NHF")) == 0);
  // symmetric J: upper blocks in the colour launches, lower ones by one
  // transpose pass (IMPM_ASM_MIRROR_PASS=0: mirrored REDs in the kernel). A
  // slab's halo nodes are not rows, so slabs keep the in-kernel mirror.
  bool mirror_pass_env = !(std::getenv("IMPM_ASM_MIRROR_PASS") && std::atoi(std::getenv("IMPM_ASM_MIRROR_PASS")) == 0);
  int last_cg_iters = 0;
  int mg_f16sim = std::getenv("IMPM_MG_F16SIM") ? std::atoi(std::getenv("IMPM_MG_F16SIM")) : 0;  // A/B experiment
  // fine-level smoother matrix in fp16 with fp32 row scales (IMPM_MG_F16=0: fp32)
  bool mg_f16 = !(std::getenv("IMPM_MG_F16") && std::atoi(std::getenv("IMPM_MG_F16")) == 0);
  // fp32 twins of the V-cycle iterates feed the fp32 level SpMV gathers
  bool mg_x4 = !(std::getenv("IMPM_MG_X4") && std::atoi(std::getenv("IMPM_MG_X4")) == 0);
  bool krylov_debug = std::getenv("IMPM_DEBUG_KRYLOV") != nullptr;
  bool res_staged = !(std::getenv("IMPM_RES_UNSTAGED") && std::atoi(std::getenv("IMPM_RES_UNSTAGED")) != 0);

  // slab decomposition along axis 0; comm == nullptr or a
  // single rank -> the plain single-GPU path
  std::shared_ptr<Comm> comm;
  bool slab = false;
  int own_lo = 0, own_hi = 0;  // owned axis-0 node range, local indices
  int glob_n0 = 0;
  std::vector<int> cuts;       // global ownership cuts [nranks + 1]
  int64_t n_dofs_glob = 0, dof_offset = 0;
  DBuf<long long> slab_counts;
  DBuf<int> mig_flag, mig_pos;
  DBuf<double> mig_send_l, mig_send_r, mig_recv_l, mig_recv_r;
  bool multi() const { return comm && comm->nranks > 1; }
  int ndg() const { return static_cast<int>(std::min<int64_t>(n_dofs_glob, INT_MAX)); }
  template <class Fn>
  void comm_call(Fn&& fn) {
    try {
      fn();
    } catch (const CommError& e) {
      throw SimError(IMPM_ERR_NCCL, e.what());
    }
  }
  // elementwise sum over ranks of reduction partials (then every rank's
  // fixed-order finalize yields the same global value)
  void gsum(double* d, size_t n) {
    if (multi()) comm_call([&] { comm->allreduce(d, n, RedType::F64, RedOp::Sum, s); });
  }
  void gmin_int(int* d, size_t n) {
    if (multi()) comm_call([&] { comm->allreduce(d, n, RedType::I32, RedOp::Min, s); });
  }
  // 2-plane halo of a grid-layout vector [node][F] along axis 0: my first /
  // last two owned planes go to the neighbours, theirs fill my halo planes
  void halo(const double* vc, int comps = -1) {
    if (!multi()) return;
    double* v = const_cast<double*>(vc);
    const size_t plane = static_cast<size_t>(g.stride[0]) * (comps > 0 ? comps : F);
    const size_t bytes = 2 * plane * sizeof(double);
    std::vector<Comm::Msg> snd, rcv;
    const int rk = comm->rank;
    if (rk > 0) {
      snd.push_back({rk - 1, v + own_lo * plane, bytes});
      rcv.push_back({rk - 1, v + (own_lo - 2) * plane, bytes});
    }
    if (rk < comm->nranks - 1) {
      snd.push_back({rk + 1, v + (own_hi - 2) * plane, bytes});
      rcv.push_back({rk + 1, v + own_hi * plane, bytes});
    }
    comm_call([&] { comm->exchange(snd, rcv, s); });
  }
  // local colour-batch start along axis 0 for GLOBAL colour c0, so slabs push
  // bins in the single-GPU batch order (bitwise-identical owned rows)
  int colour0(int c0) const { return ((c0 - g.base0) % 3 + 3) % 3; }

  // controller state (mpm_solver.hpp:466-477)
  bool step_built = false;
  bool have_prev = false;
  bool have_uwarm = false;
  int step_counter = 0;

  // last error
  std::string err_msg;
  std::vector<double> err_hist;
  Prof prof;

  int64_t NF() const { return static_cast<int64_t>(g.N) * F; }

  template <class Fn>
  void dispatch(Fn&& fn) {
    const int key_ = D * 10 + shape;
    switch (key_) {
      case 11: fn(IC<1>{}, IC<1>{}); break;
      case 12: fn(IC<1>{}, IC<2>{}); break;
      case 21: fn(IC<2>{}, IC<1>{}); break;
      case 22: fn(IC<2>{}, IC<2>{}); break;
      case 31: fn(IC<3>{}, IC<1>{}); break;
      case 32: fn(IC<3>{}, IC<2>{}); break;
      default: throw SimError(IMPM_ERR_CONFIG, "unsupported dimension/shape");
    }
  }

  template <class Fn>
  void dispatch_df(Fn&& fn) {
    switch (D * 10 + F) {
      case 11: fn(IC<1>{}, IC<1>{}); break;
      case 22: fn(IC<2>{}, IC<2>{}); break;
      case 33: fn(IC<3>{}, IC<3>{}); break;
      case 23: fn(IC<2>{}, IC<3>{}); break;
      case 34: fn(IC<3>{}, IC<4>{}); break;
      default: throw SimError(IMPM_ERR_CONFIG, "unsupported dimension/field combination");
    }
  }

  MatParams matp() const {
    MatParams m;
    m.kind = mat.kind;
    const double E = mat.E, nu = mat.nu;
    m.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));  // materials.hpp:16-17
    m.mu = E / (2.0 * (1.0 + nu));
    m.kappa = mat.kappa;
    const double sphi = std::sin(mat.friction_deg * M_PI / 180.0);
    m.dp_alpha = std::sqrt(2.0 / 3.0) * 2.0 * sphi / (3.0 - sphi);
    m.dp_ec = 3.0 * mat.cohesion / (3.0 * m.lam + 2.0 * m.mu);
    m.mcc_M = 6.0 * sphi / (3.0 - sphi);
    m.mcc_pc0 = mat.pc0;
    m.mcc_theta = mat.hardening;
    m.mcc_pt = mat.cohesion;
    return m;
  }

  Sim(const impm_grid* gr, const impm_material* m, const impm_options* o, int dev, const impm_poro* poro = nullptr) {
    D = gr->dim;
    if (D < 1 || D > 3) throw SimError(IMPM_ERR_CONFIG, "grid dimension must be 1, 2 or 3");
    F = D;
    if (poro) {
      // the reference's CoupledSim is 2D (porous.hpp:48); D = 3 (4x4 blocks) is an extension
      if (D != 2 && D != 3) throw SimError(IMPM_ERR_CONFIG, "coupled u-p requires a 2D or 3D grid");
      if (!(poro->k > 0.0)) throw SimError(IMPM_ERR_CONFIG, "permeability must be positive");  // porous.hpp:32-37
      if (!(poro->mu_f > 0.0)) throw SimError(IMPM_ERR_CONFIG, "fluid viscosity must be positive");
      if (!(poro->mu > 0.0) || !(poro->lambda + 2.0 * poro->mu > 0.0))
        throw SimError(IMPM_ERR_CONFIG, "solid moduli must give a positive constrained modulus");
      coupled = true;
      F = D + 1;
      pc.lam = poro->lambda;
      pc.mu = poro->mu;
      pc.mob = poro->k / poro->mu_f;
      pc.rho_f = poro->rho_f;
    }
    device = dev;
    CK(cudaSetDevice(device));
    int N = 1;
    for (int a = 0; a < 3; ++a) {
      g.nodes[a] = a < D ? gr->nodes[a] : 1;
      g.origin[a] = a < D ? gr->origin[a] : 0.0;
      if (g.nodes[a] < 1) throw SimError(IMPM_ERR_CONFIG, "grid node counts must be positive");
      N *= g.nodes[a];
    }
    g.stride[D - 1] = 1;
    for (int a = D - 2; a >= 0; --a) g.stride[a] = g.stride[a + 1] * g.nodes[a + 1];
    for (int a = D; a < 3; ++a) g.stride[a] = 0;
    g.h = gr->h;
    g.N = N;
    if (!(g.h > 0.0)) throw SimError(IMPM_ERR_CONFIG, "grid spacing must be positive");
    if (!coupled) set_material(m);
    set_options(o);
    CK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
    s = own_stream;
    prof.s = s;
    CK(cudaStreamCreateWithFlags(&io_stream, cudaStreamNonBlocking));
    for (auto& e : io_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    fixed.ensure(NF());
    CK(cudaMemsetAsync(fixed.p, 0, NF(), s));
    st.ensure(1);
    dflag.ensure(4);
    sc.ensure(kNSlots);
    partials.ensure(8 * kRedBlocks + kSpmvMaxBlocks);
    if (const char* e = std::getenv("IMPM_MG_F64")) mg_f32 = std::atoi(e) == 0;  // A/B experiments only
    if (const char* e = std::getenv("IMPM_MG_REUSE")) mg_reuse = std::atoi(e) != 0;
    if (const char* e = std::getenv("IMPM_ETA0_FACTOR")) newton_eta_factor = std::atof(e);  // A/B experiments
    if (const char* e = std::getenv("IMPM_EXACT_RTOL")) exact_rtol = std::atof(e);       // A/B experiments
    if (const char* e = std::getenv("IMPM_EXACT_NEWTON")) exact_newton_env = std::atoi(e);  // A/B experiments
    if (const char* e = std::getenv("IMPM_MG_SMOOTH")) mg_smooth_env = std::atoi(e);
    if (const char* e = std::getenv("IMPM_TANGENT_K1")) tangent_k1 = std::atoi(e) != 0;
    if (const char* e = std::getenv("IMPM_SPMV_BLOCKS"))  // tuning experiments only
      spmv_blocks = std::max(1, std::min(kSpmvMaxBlocks, std::atoi(e)));
    mg_blocks = spmv_blocks;
    if (const char* e = std::getenv("IMPM_MG_BLOCKS"))  // tuning experiments only
      mg_blocks = std::max(1, std::min(kSpmvMaxBlocks, std::atoi(e)));
    sums.ensure(8);
    CK(cudaMallocHost(&h_st, sizeof(DevStatus)));
    CK(cudaMallocHost(&h_sc, sizeof(double) * kNSlots));
    ND = 6 * D + 22 + D * D;
    CK(cudaStreamSynchronize(s));
  }
  ~Sim() {
    if (h_st) cudaFreeHost(h_st);
    if (h_sc) cudaFreeHost(h_sc);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (io_stream) cudaStreamDestroy(io_stream);
    for (auto& e : io_ev)
      if (e) cudaEventDestroy(e);
  }

  void set_material(const impm_material* m) {
    mat = *m;
    if (!(mat.E > 0.0)) throw SimError(IMPM_ERR_CONFIG, "Young's modulus must be positive");
    if (!(mat.nu > -1.0 && mat.nu < 0.5)) throw SimError(IMPM_ERR_CONFIG, "Poisson's ratio must lie in (-1, 0.5)");
    if (mat.kind != kHencky && mat.kind != kHenckyJ2 && mat.kind != kNeoHookean && mat.kind != kDruckerPrager &&
        mat.kind != kCamClay)
      throw SimError(IMPM_ERR_CONFIG, "unknown material kind");
    if (mat.kind == kDruckerPrager && !(mat.friction_deg > 0.0 && mat.friction_deg < 90.0))
      throw SimError(IMPM_ERR_CONFIG, "Drucker-Prager friction angle must lie in (0, 90) degrees");
    if (mat.kind == kCamClay) {
      if (!(mat.friction_deg > 0.0 && mat.friction_deg < 90.0))
        throw SimError(IMPM_ERR_CONFIG, "Cam-Clay critical-state friction angle must lie in (0, 90) degrees");
      if (!(mat.pc0 > 0.0)) throw SimError(IMPM_ERR_CONFIG, "Cam-Clay preconsolidation pressure must be positive");
      if (!(mat.hardening >= 0.0)) throw SimError(IMPM_ERR_CONFIG, "Cam-Clay hardening must be non-negative");
      if (!(mat.cohesion > 0.0)) throw SimError(IMPM_ERR_CONFIG, "Cam-Clay tensile intercept must be positive");
    }
    // the reference has Hencky / J2 only for D <= 2 (mpm_solver.hpp:448-453);
    // here every kind runs in 3D through the spectral log/exp (extension)
    if (mat.kind == kHenckyJ2 && !(mat.kappa > 0.0)) throw SimError(IMPM_ERR_CONFIG, "yield strength must be positive");
  }
  void set_options(const impm_options* o) {
    opt = *o;
    if (opt.max_iterations <= 0) opt.max_iterations = 20;
    if (!(opt.tol > 0.0)) opt.tol = 1e-11;
    if (!(opt.abs_floor >= 0.0)) opt.abs_floor = 1e-14;
    if (!(opt.krylov_rtol > 0.0)) opt.krylov_rtol = 1e-12;
    cur_rtol = opt.krylov_rtol;
    shape = opt.shape == IMPM_SHAPE_BSPLINE2 ? 2 : 1;
    if (!coupled && opt.total_lagrangian && has_history(mat.kind))  // mpm_solver.hpp:66-67
      throw SimError(IMPM_ERR_CONFIG, "total-Lagrangian stepping supports elastic materials only");
    prof.on = opt.profile != 0;
  }

  void sync() { CK(cudaStreamSynchronize(s)); }

  void reset_status() {
    DevStatus z{};
    z.err_domain = INT_MAX;
    z.err_ood = INT_MAX;
    z.err_cfg = INT_MAX;
    z.err_lp = INT_MAX;
    z.err_seed = INT_MAX;
    z.max_mass = 0.0;
    *h_st = z;
    CK(cudaMemcpyAsync(st.p, h_st, sizeof(DevStatus), cudaMemcpyHostToDevice, s));
  }
  void read_status() {
    CK(cudaMemcpyAsync(h_st, st.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
    sync();
  }
  void clear_errors_only() {
    // reset the error words, keep max_mass
    const int big = INT_MAX;
    CK(cudaMemcpyAsync(&st.p->err_domain, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  }

  // ---------------------------------------------------------- particles
  void set_particles(const double* aos, int64_t n, int64_t stride) {
    if (stride % 8 != 0 || stride < ND * 8) throw SimError(IMPM_ERR_CONFIG, "bad particle stride");
    if (n > INT_MAX / 2) throw SimError(IMPM_ERR_CONFIG, "too many particles");
    P = static_cast<int>(n);
    cap = std::max<int64_t>(P, 1);
    pd.ensure(cap * ND);
    orig.ensure(cap);
    ensure_particle_buffers();
    CK(cudaMemsetAsync(uty.p, 0, sizeof(double) * cap, s));
    DBuf<double>& staging = io_staging;  // persistent: no 3 GB malloc/free per call
    staging.ensure(std::max<int64_t>(1, n * (stride / 8)));
    const int K = stride == ND * 8 && n >= (1 << 20) ? io_chunks : 1;
    if (n > 0 && K > 1) {
      // chunk c's upload (io_stream) overlaps chunk c-1's transpose (s)
      const int64_t ch = (n + K - 1) / K;
      CK(cudaEventRecord(io_ev[kIoMaxChunks], s));  // staging is free once s got here
      CK(cudaStreamWaitEvent(io_stream, io_ev[kIoMaxChunks], 0));
      for (int c = 0; c < K; ++c) {
        const int64_t r0 = c * ch, r1 = std::min<int64_t>(n, r0 + ch);
        if (r0 >= r1) break;
        CK(cudaMemcpyAsync(staging.p + r0 * ND, aos + r0 * ND, (r1 - r0) * stride, cudaMemcpyHostToDevice, io_stream));
        CK(cudaEventRecord(io_ev[c], io_stream));
        CK(cudaStreamWaitEvent(s, io_ev[c], 0));
        k_aos_rows_to_soa<<<blocks_for(r1 - r0), kThreads, 0, s>>>(staging.p, static_cast<int>(r0),
                                                                     static_cast<int>(r1), ND, pd.p, cap, orig.p);
        ++g_launches;
        CKL();
      }
    } else if (n > 0) {
      CK(cudaMemcpyAsync(staging.p, aos, n * stride, cudaMemcpyHostToDevice, s));
      k_aos_to_soa<<<blocks_for(n), kThreads, 0, s>>>(staging.p, stride / 8, P, ND, pd.p, cap, orig.p); ++g_launches;
      CKL();
    }
    sync();
    step_built = false;
    matrix_valid = false;
    f16_ready = false;
  }
  // per-particle work arrays sized by `cap` (the SoA field stride)
  void ensure_particle_buffers() {
    pd_tmp.ensure(cap * ND);
    xs.ensure(cap * 3);
    bext.ensure(cap * 3);
    orig_tmp.ensure(cap);
    key.ensure(cap);
    sup.ensure(cap);
    rank.ensure(cap);
    perm.ensure(cap);
    Pst.ensure(cap * (D * D + 2 + D));  // single field: D*D; u-p: UpQ<D>::N
    uty.ensure(cap);
    Atan.ensure(cap * D * D * D * D);
  }
  void get_particles(double* aos, int64_t n, int64_t stride) {
    if (slab) throw SimError(IMPM_ERR_UNSUPPORTED, "a slab holds a subset of the particles: use get_particles_ids");
    if (n != P) throw SimError(IMPM_ERR_CONFIG, "particle count mismatch");
    if (stride % 8 != 0 || stride < ND * 8) throw SimError(IMPM_ERR_CONFIG, "bad particle stride");
    if (n == 0) return;
    DBuf<double>& staging = io_staging;
    staging.ensure(n * (stride / 8));
    const int K = stride == ND * 8 && n >= (1 << 20) ? io_chunks : 1;
    if (K > 1) {
      // rows in original order, chunk by chunk: chunk c's download
      // (io_stream) overlaps chunk c+1's gather (s)
      io_inv.ensure(n);
      k_invert_perm<<<blocks_for(n), kThreads, 0, s>>>(orig.p, P, io_inv.p); ++g_launches;
      const int64_t ch = (n + K - 1) / K;
      for (int c = 0; c < K; ++c) {
        const int64_t o0 = c * ch, o1 = std::min<int64_t>(n, o0 + ch);
        if (o0 >= o1) break;
        k_rows_to_aos<<<148 * 8, kThreads, 0, s>>>(pd.p, cap, io_inv.p, static_cast<int>(o0), static_cast<int>(o1), ND,
                                                   staging.p);
        ++g_launches;
        CKL();
        CK(cudaEventRecord(io_ev[c], s));
        CK(cudaStreamWaitEvent(io_stream, io_ev[c], 0));
        CK(cudaMemcpyAsync(aos + o0 * ND, staging.p + o0 * ND, (o1 - o0) * stride, cudaMemcpyDeviceToHost, io_stream));
      }
      CK(cudaStreamSynchronize(io_stream));
      sync();
      return;
    }
    if (stride != ND * 8) CK(cudaMemcpyAsync(staging.p, aos, n * stride, cudaMemcpyHostToDevice, s));
    k_soa_to_aos<<<blocks_for(n), kThreads, 0, s>>>(pd.p, cap, P, ND, orig.p, staging.p, stride / 8); ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(aos, staging.p, n * stride, cudaMemcpyDeviceToHost, s));
    sync();
  }
  // slab particles carry their global ids (= the single-GPU AoS index), used
  // for error messages and as the identity of migrated particles
  void set_particles_ids(const double* aos, const int64_t* ids, int64_t n, int64_t stride) {
    set_particles(aos, n, stride);
    if (n == 0) return;
    std::vector<int> h(n);
    for (int64_t i = 0; i < n; ++i) {
      if (ids[i] < 0 || ids[i] > INT_MAX / 4) throw SimError(IMPM_ERR_CONFIG, "particle ids must lie in [0, 2^29)");
      h[i] = static_cast<int>(ids[i]);
    }
    CK(cudaMemcpyAsync(orig.p, h.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    sync();
  }
  // local particles (owned + ghost copies) in local order, with global ids
  void get_particles_ids(double* aos, int64_t* ids, int64_t n, int64_t stride) {
    if (n != P) throw SimError(IMPM_ERR_CONFIG, "particle count mismatch");
    if (stride % 8 != 0 || stride < ND * 8) throw SimError(IMPM_ERR_CONFIG, "bad particle stride");
    if (n == 0) return;
    DBuf<double>& staging = io_staging;
    DBuf<long long> dids;
    staging.ensure(n * (stride / 8));
    dids.ensure(n);
    if (stride != ND * 8) CK(cudaMemsetAsync(staging.p, 0, n * stride, s));
    k_soa_to_aos_ids<<<blocks_for(n), kThreads, 0, s>>>(pd.p, cap, P, ND, orig.p, staging.p, stride / 8, dids.p);
    ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(aos, staging.p, n * stride, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ids, dids.p, sizeof(long long) * n, cudaMemcpyDeviceToHost, s));
    sync();
  }

  // ---------------------------------------------------- slab decomposition
  // The caller creates the Sim on the LOCAL grid: global origin, nodes[0] =
  // hi - lo with [lo, hi) = [max(0, A - 2), min(n0, B + 2)) for the owned
  // planes [A, B) = [cuts[rank], cuts[rank + 1]).
  void set_slab(std::shared_ptr<Comm> c, int n0, const int* cuts_in) {
    if (coupled) throw SimError(IMPM_ERR_UNSUPPORTED, "slab decomposition supports the single-field MpmSim only");
    const int nr = c->nranks, rk = c->rank;
    std::vector<int> cu(cuts_in, cuts_in + nr + 1);
    if (cu[0] != 0 || cu[nr] != n0) throw SimError(IMPM_ERR_CONFIG, "slab cuts must span [0, n0]");
    for (int q = 0; q < nr; ++q)
      if (cu[q + 1] - cu[q] < (nr > 1 ? 4 : 1))
        throw SimError(IMPM_ERR_CONFIG, "every slab needs at least 4 owned node planes along axis 0");
    const int lo = std::max(0, cu[rk] - 2), hi = std::min(n0, cu[rk + 1] + 2);
    if (g.nodes[0] != hi - lo)
      throw SimError(IMPM_ERR_CONFIG, "slab grid must hold the owned planes plus a 2-plane halo: nodes[0] = " +
                                          std::to_string(hi - lo));
    g.base0 = lo;
    own_lo = cu[rk] - lo;
    own_hi = cu[rk + 1] - lo;
    glob_n0 = n0;
    cuts = cu;
    comm = std::move(c);
    slab = true;
    step_built = false;
    matrix_valid = false;
    f16_ready = false;
  }

  // After commit_step: every owned particle goes to the rank(s) that keep it
  // for the next step (owner + the neighbour that needs it as a ghost),
  // ghost copies are dropped; the new local array is [from left | kept |
  // from right], i.e. the global sorted order restricted to this slab, so
  // the stable bin sort reproduces the single-GPU particle order per bin.
  void migrate() {
    if (!slab) throw SimError(IMPM_ERR_CONFIG, "migrate on a simulation without a slab decomposition");
    if (!multi() || opt.total_lagrangian) return;  // TL supports never move (support on X)
    const int rk = comm->rank, nr = comm->nranks;
    const bool hl = rk > 0, hr = rk < nr - 1;
    const int A = cuts[rk], B = cuts[rk + 1];
    const int lo_ok = hl ? cuts[rk - 1] : INT_MIN;
    const int hi_ok = hr ? (rk + 2 < nr ? cuts[rk + 2] - 2 : glob_n0) : INT_MAX;
    mig_flag.ensure(3 * cap);
    mig_pos.ensure(3 * (cap + 1));
    int* fk = mig_flag.p;
    int* fl = mig_flag.p + cap;
    int* fr = mig_flag.p + 2 * cap;
    int* pk = mig_pos.p;
    int* pl = mig_pos.p + (cap + 1);
    int* pr = mig_pos.p + 2 * (cap + 1);
    const int big = INT_MAX;
    CK(cudaMemcpyAsync(&st.p->err_migrate, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    if (P > 0) {
      dispatch([&](auto Dc, auto Sc) {
        constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
        k_migrate_flags<DD, SH><<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, g, key.p, 0, own_lo, own_hi, A, B,
                                                                    hl, hr, lo_ok, hi_ok, orig.p, fk, fl, fr, st.p);
        ++g_launches;
        CKL();
      });
    }
    scan<int>(fk, P, pk, scan_sums_i, pk + P);
    scan<int>(fl, P, pl, scan_sums_i, pl + P);
    scan<int>(fr, P, pr, scan_sums_i, pr + P);
    gmin_int(&st.p->err_migrate, 1);
    int cnt[3];
    CK(cudaMemcpyAsync(&cnt[0], pk + P, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&cnt[1], pl + P, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&cnt[2], pr + P, sizeof(int), cudaMemcpyDeviceToHost, s));
    read_status();
    if (h_st->err_migrate != INT_MAX)
      throw SimError(IMPM_ERR_DOMAIN, "particle " + std::to_string(h_st->err_migrate) +
                                          " moved past the neighbouring slab in one step");
    if (P == 0) cnt[0] = cnt[1] = cnt[2] = 0;
    const int nk = cnt[0], nl = cnt[1], nrr = cnt[2];
    // counts, then payloads (records of ND doubles + id)
    slab_counts.ensure(4);
    long long hc[4] = {nl, nrr, 0, 0};
    CK(cudaMemcpyAsync(slab_counts.p, hc, sizeof(hc), cudaMemcpyHostToDevice, s));
    {
      std::vector<Comm::Msg> snd, rcv;
      if (hl) {
        snd.push_back({rk - 1, slab_counts.p + 0, sizeof(long long)});
        rcv.push_back({rk - 1, slab_counts.p + 2, sizeof(long long)});
      }
      if (hr) {
        snd.push_back({rk + 1, slab_counts.p + 1, sizeof(long long)});
        rcv.push_back({rk + 1, slab_counts.p + 3, sizeof(long long)});
      }
      comm_call([&] { comm->exchange(snd, rcv, s); });
    }
    CK(cudaMemcpyAsync(hc, slab_counts.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    sync();
    const int cl = static_cast<int>(hc[2]), cr = static_cast<int>(hc[3]);
    const int RW = ND + 1;
    mig_send_l.ensure(static_cast<size_t>(std::max(nl, 1)) * RW);
    mig_send_r.ensure(static_cast<size_t>(std::max(nrr, 1)) * RW);
    mig_recv_l.ensure(static_cast<size_t>(std::max(cl, 1)) * RW);
    mig_recv_r.ensure(static_cast<size_t>(std::max(cr, 1)) * RW);
    if (P > 0) {
      k_pack_records<<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, ND, orig.p, fl, pl, mig_send_l.p); ++g_launches;
      k_pack_records<<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, ND, orig.p, fr, pr, mig_send_r.p); ++g_launches;
      CKL();
    }
    {
      std::vector<Comm::Msg> snd, rcv;
      const size_t rb = sizeof(double) * RW;
      if (hl) {
        snd.push_back({rk - 1, mig_send_l.p, rb * nl});
        rcv.push_back({rk - 1, mig_recv_l.p, rb * cl});
      }
      if (hr) {
        snd.push_back({rk + 1, mig_send_r.p, rb * nrr});
        rcv.push_back({rk + 1, mig_recv_r.p, rb * cr});
      }
      comm_call([&] { comm->exchange(snd, rcv, s); });
    }
    const int newP = cl + nk + cr;
    // grow with headroom: every growth reallocates all per-particle buffers
    const int64_t newcap = newP > cap ? newP + newP / 32 + 1 : cap;
    pd_tmp.ensure(newcap * ND);
    orig_tmp.ensure(newcap);
    if (cl > 0) {
      k_unpack_records<<<blocks_for(cl), kThreads, 0, s>>>(mig_recv_l.p, cl, ND, pd_tmp.p, newcap, 0, orig_tmp.p);
      ++g_launches;
    }
    if (P > 0) {
      k_keep_gather<<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, ND, orig.p, fk, pk, pd_tmp.p, newcap, cl,
                                                       orig_tmp.p);
      ++g_launches;
    }
    if (cr > 0) {
      k_unpack_records<<<blocks_for(cr), kThreads, 0, s>>>(mig_recv_r.p, cr, ND, pd_tmp.p, newcap, cl + nk,
                                                           orig_tmp.p);
      ++g_launches;
    }
    CKL();
    std::swap(pd.p, pd_tmp.p);
    std::swap(pd.cap, pd_tmp.cap);
    std::swap(orig.p, orig_tmp.p);
    std::swap(orig.cap, orig_tmp.cap);
    P = newP;
    cap = newcap;
    ensure_particle_buffers();
    sync();
    step_built = false;
    matrix_valid = false;
    f16_ready = false;
  }

  void set_particle_field(int field, const double* vals_h) {
    if (slab) throw SimError(IMPM_ERR_UNSUPPORTED, "set_particle_field indexes the full particle set");
    if (field < 0 || field >= ND) throw SimError(IMPM_ERR_CONFIG, "bad particle field");
    DBuf<double> tmp;
    tmp.ensure(std::max(P, 1));
    CK(cudaMemcpyAsync(tmp.p, vals_h, sizeof(double) * P, cudaMemcpyHostToDevice, s));
    k_set_field<<<blocks_for(P), kThreads, 0, s>>>(pd.p + field * cap, tmp.p, orig.p, P); ++g_launches;
    CKL();
    sync();
    step_built = false;
  }

  // ---------------------------------------------------------- scans
  template <class T>
  void scan(const int* in, int64_t n, T* out, DBuf<T>& sums_buf, T* total_slot) {
    const int64_t nb = (n + 4095) / 4096;
    sums_buf.ensure(nb + 1);
    k_scan_block<T><<<static_cast<unsigned>(std::max<int64_t>(nb, 1)), 1024, 0, s>>>(in, n, out, sums_buf.p); ++g_launches;
    CKL();
    k_scan_sums<T><<<1, 1024, 0, s>>>(sums_buf.p, static_cast<int>(nb), sums_buf.p + nb); ++g_launches;
    CKL();
    k_scan_add<T><<<blocks_for(std::max<int64_t>(n, 1)), kThreads, 0, s>>>(out, n, sums_buf.p, sums_buf.p + nb,
                                                                           total_slot); ++g_launches;
    CKL();
  }

  // active rows in brick-major order (see k_brick_flags); returns n_act
  template <int DD>
  void brick_rows(const GridC& gg, const int* act_flag_p, int* act_idx_p, int* act_list_p, int* n_out_dev) {
    int64_t nb = 1;
    for (int a = 0; a < DD; ++a) nb *= (gg.nodes[a] + 3) / 4;
    nb <<= 2 * DD;
    brick_flag.ensure(nb);
    brick_scan.ensure(nb + 1);
    CK(cudaMemsetAsync(brick_flag.p, 0, sizeof(int) * nb, s));
    k_brick_flags<DD><<<blocks_for(gg.N), kThreads, 0, s>>>(gg, act_flag_p, brick_flag.p); ++g_launches;
    CKL();
    scan<int>(brick_flag.p, nb, brick_scan.p, scan_sums_i, brick_scan.p + nb);
    k_act_finalize_brick<DD><<<blocks_for(gg.N), kThreads, 0, s>>>(gg, act_flag_p, brick_scan.p, act_idx_p,
                                                                    act_list_p); ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(n_out_dev, brick_scan.p + nb, sizeof(int), cudaMemcpyDeviceToDevice, s));
  }

  // ------------------------------------------------- begin_step (K1-K4)
  std::string ood_message(int code) {
    return "particle " + std::to_string(code / 4) + " has support outside the grid on axis " +
           std::to_string(code % 4);
  }

  void begin_step() {
    ref_nnz_cache = -1;  // the pattern follows this step's DOF map
    if ((opt.total_lagrangian || coupled) && step_built) return;  // mpm_solver.hpp:94, porous.cpp:92
    const int N = g.N;
    reset_status();
    bin_count.ensure(N + 1);
    bin_start.ensure(N + 1);
    mass.ensure(N);
    act_flag.ensure(N);
    act_scan.ensure(N + 1);
    act_idx.ensure(N);
    act_list.ensure(N);
    free_flag.ensure(NF());
    free_scan.ensure(NF() + 1);
    freem.ensure(NF());
    dof_of.ensure(NF());
    node_of.ensure(NF());
    field_of.ensure(NF());
    for (auto* v : {&u, &r, &delta, &utry, &rtry, &prev, &tmp1, &tmp2, &kx, &kr, &kz, &kp, &kq, &kv, &ks, &kt, &khat})
      v->ensure(NF());
    // work vectors are only ever written at active rows: keep the rest zero
    for (auto* v : {&delta, &utry, &rtry, &tmp1, &tmp2, &kx, &kr, &kz, &kp, &kq, &kv, &ks, &kt, &khat})
      CK(cudaMemsetAsync(v->p, 0, sizeof(double) * NF(), s));
    {
      Prof::Scope ps(&prof, kcSort);
      dispatch([&](auto Dc, auto Sc) {
        constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
        if (P > 0) {
          k_support<DD, SH><<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, g, orig.p, key.p, sup.p, xs.p, st.p,
                                                                coupled ? 1 : 0); ++g_launches;
          CKL();
        }
      });
    }
    gmin_int(&st.p->err_domain, 3);  // err_domain, err_ood, err_cfg
    read_status();
    if (h_st->err_ood != INT_MAX) throw SimError(IMPM_ERR_OUT_OF_DOMAIN, ood_message(h_st->err_ood));
    if (h_st->err_cfg != INT_MAX)
      throw SimError(IMPM_ERR_CONFIG, "GIMP requires 0 < lp < h/2 (particle " + std::to_string(h_st->err_cfg) + ")");
    // SolverOptions::interference (mpm_solver.hpp:31, jacobian.hpp:126-128):
    // the supports fix every Jacobian of the step, so the check runs here
    if (opt.interference != IMPM_INTERFERENCE_OFF && h_st->err_seed != INT_MAX) {
      const int pid = h_st->err_seed / 4, ax = h_st->err_seed % 4;
      throw SimError(IMPM_ERR_SEEDING, "backward pass touched a dof outside every seeded pattern of its group "
                                       "(particle " + std::to_string(pid) + " spans more than 3 nodes on axis " +
                                       std::to_string(ax) + ")");
    }
    {
      Prof::Scope ps(&prof, kcSort);
      // counting sort by first support node (K1)
      CK(cudaMemsetAsync(bin_count.p, 0, sizeof(int) * (N + 1), s));
      if (P > 0) {
        k_bin_count<<<blocks_for(P), kThreads, 0, s>>>(key.p, P, bin_count.p, rank.p); ++g_launches;
        CKL();
      }
      scan<int>(bin_count.p, N, bin_start.p, scan_sums_i, bin_start.p + N);
      if (P > 0) {
        k_bin_scatter<<<blocks_for(P), kThreads, 0, s>>>(key.p, rank.p, bin_start.p, P, perm.p); ++g_launches;
        CKL();
        k_bin_sort<<<blocks_for(N), kThreads, 0, s>>>(bin_start.p, N, perm.p); ++g_launches;
        CKL();
        k_perm_check<<<blocks_for(P), kThreads, 0, s>>>(perm.p, P, st.p); ++g_launches;
        CKL();
      }
    }
    read_status();
    if (h_st->perm_moved) {
      Prof::Scope ps(&prof, kcSort);
      constexpr int kFpb = 8;  // fields per thread
      dim3 grid(blocks_for(P), (ND + kFpb - 1) / kFpb);
      k_gather_fields<<<grid, kThreads, 0, s>>>(pd.p, pd_tmp.p, cap, perm.p, P, ND, kFpb); ++g_launches;
      CKL();
      k_gather_int<<<blocks_for(P), kThreads, 0, s>>>(orig.p, orig_tmp.p, perm.p, P); ++g_launches;
      k_gather_fields<<<dim3(blocks_for(P), 1), kThreads, 0, s>>>(uty.p, xs.p, cap, perm.p, P); ++g_launches;
      CK(cudaMemcpyAsync(uty.p, xs.p, sizeof(double) * P, cudaMemcpyDeviceToDevice, s));
      CKL();
      std::swap(pd.p, pd_tmp.p);
      std::swap(pd.cap, pd_tmp.cap);
      std::swap(orig.p, orig_tmp.p);
      std::swap(orig.cap, orig_tmp.cap);
      dispatch([&](auto Dc, auto Sc) {
        constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
        k_support<DD, SH><<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, g, orig.p, key.p, sup.p, xs.p, st.p,
                                                                coupled ? 1 : 0); ++g_launches;
        CKL();
      });
    }
    {
      Prof::Scope ps(&prof, kcMass);
      dispatch([&](auto Dc, auto Sc) {
        constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
        if (P > 0) {
          k_bext<DD><<<blocks_for(P), kThreads, 0, s>>>(pd.p, cap, P, gravity[0], gravity[1], gravity[2], bext.p, st.p); ++g_launches;
          CKL();
        }
        // activity cutoff 1e-12 * max particle mass over ALL particles
        if (multi()) comm_call([&] { comm->allreduce(&st.p->max_mass, 1, RedType::F64, RedOp::Max, s); });
        if (coupled) {
          if constexpr (DD == 2)
            k_node_mass<2, 3, SH><<<blocks_for(N), kThreads, 0, s>>>(g, pd.p, cap, xs.p, bin_start.p, sup.p, fixed.p,
                                                                      st.p, mass.p, act_flag.p, free_flag.p);
          else if constexpr (DD == 3)
            k_node_mass<3, 4, SH><<<blocks_for(N), kThreads, 0, s>>>(g, pd.p, cap, xs.p, bin_start.p, sup.p, fixed.p,
                                                                      st.p, mass.p, act_flag.p, free_flag.p);
        } else {
          k_node_mass<DD, DD, SH><<<blocks_for(N), kThreads, 0, s>>>(g, pd.p, cap, xs.p, bin_start.p, sup.p, fixed.p,
                                                                      st.p, mass.p, act_flag.p, free_flag.p);
        } ++g_launches;
        CKL();
        if (slab) {
          k_mask_owned<<<blocks_for(N), kThreads, 0, s>>>(N, F, g.stride[0], own_lo, own_hi, act_flag.p, free_flag.p);
          ++g_launches;
          CKL();
        }
      });
    }
    {
      Prof::Scope ps(&prof, kcDof);
      scan<int>(free_flag.p, NF(), free_scan.p, scan_sums_i, free_scan.p + NF());
      k_dof_finalize<<<blocks_for(NF()), kThreads, 0, s>>>(static_cast<int>(NF()), F, free_flag.p, free_scan.p,
                                                             dof_of.p, node_of.p, field_of.p, freem.p); ++g_launches;
      CKL();
      dispatch([&](auto Dc, auto) {
        constexpr int DD = decltype(Dc)::value;
        brick_rows<DD>(g, act_flag.p, act_idx.p, act_list.p, act_scan.p + N);
      });
    }
    int counts[2];
    CK(cudaMemcpyAsync(&counts[0], free_scan.p + NF(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&counts[1], act_scan.p + N, sizeof(int), cudaMemcpyDeviceToHost, s));
    sync();
    prof.flush();
    n_dofs = counts[0];
    n_act = counts[1];
    // global DofMap = exclusive scan of the owned free-DOF counts in rank
    // order (grid.hpp:69-86 numbers nodes in ascending flat order, axis 0
    // slowest, so each slab's DOFs are one contiguous global range)
    n_dofs_glob = n_dofs;
    dof_offset = 0;
    if (multi()) {
      const int nr = comm->nranks;
      slab_counts.ensure(std::max(nr, 4));
      std::vector<long long> hcnt(nr, 0);
      hcnt[comm->rank] = n_dofs;
      CK(cudaMemcpyAsync(slab_counts.p, hcnt.data(), sizeof(long long) * nr, cudaMemcpyHostToDevice, s));
      comm_call([&] { comm->allreduce(slab_counts.p, nr, RedType::I64, RedOp::Sum, s); });
      CK(cudaMemcpyAsync(hcnt.data(), slab_counts.p, sizeof(long long) * nr, cudaMemcpyDeviceToHost, s));
      sync();
      n_dofs_glob = 0;
      for (int q = 0; q < nr; ++q) {
        if (q < comm->rank) dof_offset += hcnt[q];
        n_dofs_glob += hcnt[q];
      }
    }
    const int S = ipow_c(5, D);
    row_len = row_len_for(S, F);
    vals.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * row_len));
    dinv.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * F * F));
    row_slots.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * S));
    row_nzb.ensure(std::max(1, n_act));
    row_mask.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * 4));
    bflag.ensure(N);
    nzb_total.ensure(1);
    {
      // Jacobian sparsity structure of this step (independent of u)
      Prof::Scope ps(&prof, kcDof);
      k_bin_flags<<<blocks_for(N), kThreads, 0, s>>>(N, D, bin_start.p, sup.p, bflag.p); ++g_launches;
      CK(cudaMemsetAsync(nzb_total.p, 0, sizeof(unsigned long long), s));
      if (n_act > 0) {
        dispatch([&](auto Dc, auto) {
          constexpr int DD = decltype(Dc)::value;
          k_row_structure<DD><<<blocks_for(n_act), kThreads, 0, s>>>(g, act_list.p, n_act, bflag.p, row_slots.p,
                                                                      row_nzb.p, row_mask.p, nzb_total.p);
          ++g_launches;
        });
      }
      CKL();
      CK(cudaMemcpyAsync(&h_nzb_total, nzb_total.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaMemsetAsync(u.p, 0, sizeof(double) * NF(), s));
    if (coupled) CK(cudaMemsetAsync(prev.p, 0, sizeof(double) * NF(), s));  // p_nodes_ = 0 (porous.cpp:70)
    matrix_valid = false;
    f16_ready = false;
    step_built = true;
    if (mg_refresh <= 1) mg_setup_step = -1;  // new row structure: rebuild the MG hierarchy
    sync();
  }

  // ------------------------------------------------------ residual (K5)
  // r = r(u) in grid layout; returns ||r||; throws DomainError on det <= 0
  double residual_dev(const double* ud, double load_scale, double* rd) {
    clear_errors_only();
    if (coupled) return residual_up(ud, load_scale, rd);
    halo(ud);
    const MatParams mp = matp();
    dispatch([&](auto Dc, auto Sc) {
      constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
      if (P > 0) {
        Prof::Scope ps(&prof, kcResP);
        if (mp.kind == kNeoHookean)
          k_residual_particles<DD, SH, true><<<blocks_for(P), kThreads, 0, s>>>(
              g, pd.p, cap, P, xs.p, key.p, sup.p, orig.p, ud, mp, opt.total_lagrangian, Pst.p, st.p);
        else
          k_residual_particles<DD, SH, false><<<blocks_for(P), kThreads, 0, s>>>(
              g, pd.p, cap, P, xs.p, key.p, sup.p, orig.p, ud, mp, opt.total_lagrangian, Pst.p, st.p);
        ++g_launches;
        CKL();
      }
      {
        Prof::Scope ps(&prof, kcResN);
        CK(cudaMemsetAsync(rd, 0, sizeof(double) * NF(), s));
        constexpr int W = 4;
        const int nc = ipow_c(3, DD);
        for (int col = 0; col < nc; ++col) {
          int cc[3] = {0, 0, 0}, nb[3] = {1, 1, 1}, rr = col;
          for (int a = DD - 1; a >= 0; --a) {
            cc[a] = a == 0 ? colour0(rr % 3) : rr % 3;
            rr /= 3;
            nb[a] = std::max(0, (g.nodes[a] - cc[a] + 2) / 3);
          }
          const int nbins = nb[0] * nb[1] * nb[2];
          if (nbins == 0) continue;
          if (res_staged)
            k_residual_bins_staged<DD, SH, W, 16><<<std::min<unsigned>(blocks_for(nbins, W), 148 * 16), W * 32, 0, s>>>(
                g, pd.p, cap, xs.p, bin_start.p, bflag.p, Pst.p, bext.p, load_scale, rd, cc[0], cc[1], cc[2], nb[0],
                nb[1], nb[2]);
          else
            k_residual_bins<DD, SH, W><<<std::min<unsigned>(blocks_for(nbins, W), 148 * 16), W * 32, 0, s>>>(
                g, pd.p, cap, xs.p, bin_start.p, bflag.p, Pst.p, bext.p, load_scale, rd, cc[0], cc[1], cc[2], nb[0],
                nb[1], nb[2]);
          ++g_launches;
        }
        k_mask_norm<<<kRedBlocks, kThreads, 0, s>>>(NF(), freem.p, rd, partials.p); ++g_launches;
        CKL();
        gsum(partials.p, kRedBlocks);
        k_finalize_sum<1><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, &st.p->norm2); ++g_launches;
        CKL();
      }
    });
    gmin_int(&st.p->err_domain, 1);
    read_status();
    prof.flush();
    if (h_st->err_domain != INT_MAX)
      throw SimError(IMPM_ERR_DOMAIN, "non-positive det(F) at particle " + std::to_string(h_st->err_domain));
    return std::sqrt(h_st->norm2);
  }

  // ------------------------------------------------------ Jacobian (K6)
  // the factored 3D neo-Hookean path (k_tangent_nh3q + k_assemble_nh3f)
  bool nhf_path(const MatParams& mp) const {
    return D == 3 && mp.kind == kNeoHookean && tangent_analytic && asm_nhf && asm_sym && !asm_rmw;
  }
  void jacobian_dev(const double* ud) {
    if (coupled) return jacobian_up(ud, up_dt);
    halo(ud);
    const MatParams mp = matp();
    dispatch([&](auto Dc, auto Sc) {
      constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
      if (P > 0) {
        Prof::Scope ps(&prof, kcTangent);
        constexpr int K = DD == 3 ? 3 : DD * DD;
        // plastic kinds (one return map per pass) take K = 3 directions per pass in 3D
        const bool nho = mp.kind == kNeoHookean;
        if (DD == 3 && nhf_path(mp))
          k_tangent_nh3q<SH><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, ud, mp,
                                                                opt.total_lagrangian, Atan.p);
        else if (DD == 3 && nho && tangent_analytic)
          k_tangent_nh3<SH><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, ud, mp,
                                                               opt.total_lagrangian, Atan.p);
        else if (DD == 3 && tangent_k1 && nho)
          k_tangent<DD, SH, 1, true><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, ud, mp,
                                                                        opt.total_lagrangian, Atan.p);
        else if (nho)
          k_tangent<DD, SH, K, true><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, ud, mp,
                                                                        opt.total_lagrangian, Atan.p);
        else
          k_tangent<DD, SH, K, false><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, ud, mp,
                                                                         opt.total_lagrangian, Atan.p);
        ++g_launches;
        CKL();
      }
      if (n_act > 0) {
        Prof::Scope ps(&prof, kcAssemble);
        const bool upper_only = asm_sym && mirror_pass_env && !multi() && !asm_rmw &&
                                mat.kind != kDruckerPrager && mat.kind != kCamClay;
        k_zero_rows<<<blocks_for(static_cast<int64_t>(n_act) * 32), kThreads, 0, s>>>(
            n_act, DD, row_nzb.p, vals.p, row_len, upper_only ? row_mask.p : nullptr, (ipow_c(5, DD) - 1) / 2);
        ++g_launches;
        constexpr int W = 4;
        constexpr int PPL = DD == 3 ? 5 : (DD == 2 ? 3 : 1);
#ifndef IMPM_ASM_PPL3
#define IMPM_ASM_PPL3 2  // 3D block pairs per lane (B200 cfg 4, ms per Jacobian: 2: 21.7, 3: 23.1, 4: 27.7)
#endif
        constexpr int asm_ppl3 = IMPM_ASM_PPL3;
        const int nc = ipow_c(3, DD);
        for (int col = 0; col < nc; ++col) {
          int cc[3] = {0, 0, 0}, nb[3] = {1, 1, 1}, r = col;
          for (int a = DD - 1; a >= 0; --a) {
            cc[a] = a == 0 ? colour0(r % 3) : r % 3;
            r /= 3;
            nb[a] = std::max(0, (g.nodes[a] - cc[a] + 2) / 3);
          }
          const int nbins = nb[0] * nb[1] * nb[2];
          if (nbins == 0) continue;
          // 3D: 4 warps of 8-particle resident bins (47.5 KB static shared, 4 CTAs/SM)
          constexpr int WS = 4;
          constexpr int PCH = DD == 3 ? 8 : 4;
          const unsigned grid = std::min<unsigned>(blocks_for(nbins, WS), 148 * 32);
          // J is symmetric except under non-associative Drucker-Prager flow and
          // Cam-Clay (associative, but its compaction hardening breaks major
          // symmetry of dP/dG: ~2% in tests/test_math_cpu.py terms)
          constexpr int PP = DD == 3 ? asm_ppl3 : PPL;
          const bool sym = asm_sym && mat.kind != kDruckerPrager && mat.kind != kCamClay;
          const bool mirror_pass = mirror_pass_env && !multi();
          auto launch = [&](auto kern, bool rmw) {
            const size_t dyn = rmw ? WS * sizeof(AsmFlush<PP, DD * DD>) : 0;
            if (rmw) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
            kern<<<grid, WS * 32, dyn, s>>>(g, pd.p, cap, xs.p, bin_start.p, bflag.p, Atan.p, act_idx.p, row_mask.p,
                                            row_nzb.p, vals.p, row_len, cc[0], cc[1], cc[2], nb[0], nb[1], nb[2]);
          };
          if constexpr (DD == 3) {
            if (nhf_path(mp)) {
              constexpr int WF = IMPM_ASMF_WARPS;
              const unsigned gridf = static_cast<unsigned>(std::min(nbins, 148 * 32));
              if (mirror_pass)
                k_assemble_nh3f<SH, WF, 8, false><<<gridf, WF * 32, 0, s>>>(
                    g, pd.p, cap, xs.p, bin_start.p, bflag.p, Atan.p, act_idx.p, row_mask.p, row_nzb.p, vals.p,
                    row_len, cc[0], cc[1], cc[2], nb[0], nb[1], nb[2]);
              else
                k_assemble_nh3f<SH, WF, 8, true><<<gridf, WF * 32, 0, s>>>(
                    g, pd.p, cap, xs.p, bin_start.p, bflag.p, Atan.p, act_idx.p, row_mask.p, row_nzb.p, vals.p,
                    row_len, cc[0], cc[1], cc[2], nb[0], nb[1], nb[2]);
              ++g_launches;
              continue;
            }
          }
          if (asm_rmw) {
            if (sym)
              launch(k_assemble_bins_staged<DD, SH, PP, WS, PCH, true, true>, true);
            else
              launch(k_assemble_bins_staged<DD, SH, PP, WS, PCH, false, true>, true);
          } else if (sym && mirror_pass) {
            launch(k_assemble_bins_staged<DD, SH, PP, WS, PCH, true, false, false>, false);
          } else if (sym) {
            launch(k_assemble_bins_staged<DD, SH, PP, WS, PCH, true, false>, false);
          } else {
            launch(k_assemble_bins_staged<DD, SH, PP, WS, PCH, false, false>, false);
          }
          ++g_launches;
        }
        f16_ready = false;
        if (upper_only) {
          if (mirror_f16 && mg_f16 && !coupled) {
            // the transpose pass also writes the MG fine level's fp16 copy
            const int64_t rl16 = row_len_of<__half>(ipow_c(5, DD), DD);
            vals16.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * rl16));
            rscale16.ensure(std::max(1, n_act));
            k_mirror_lower<DD, true><<<static_cast<unsigned>((n_act + 7) / 8), 256, 0, s>>>(
                g, n_act, act_list.p, act_idx.p, row_nzb.p, row_slots.p, row_mask.p, vals.p, row_len, vals16.p, rl16,
                rscale16.p);
            f16_ready = true;
          } else {
            k_mirror_lower<DD><<<static_cast<unsigned>((n_act + 7) / 8), 256, 0, s>>>(
                g, n_act, act_list.p, act_idx.p, row_nzb.p, row_slots.p, row_mask.p, vals.p, row_len);
          }
          ++g_launches;
          CKL();
        }
        k_diag_inverse<DD><<<blocks_for(n_act), kThreads, 0, s>>>(n_act, act_list.p, freem.p, row_mask.p, row_nzb.p,
                                                                   vals.p, row_len, dinv.p); ++g_launches;
        CKL();
      }
    });
    matrix_valid = true;
  }

  // ------------------------------------------------------- Krylov (K7)
  void spmv(const double* x, double* y, const double* dotv, double* parts) {
    halo(x);  // columns of owned rows reach 2 planes into the neighbours
    Prof::Scope ps(&prof, kcSpmv);
    dispatch_df([&](auto Dc, auto Fc) {
      constexpr int DD = decltype(Dc)::value, FE = decltype(Fc)::value;
      constexpr int W = 4;
      k_spmv<DD, FE, W><<<spmv_blocks, W * 32, 0, s>>>(g, act_list.p, n_act, vals.p, row_len, row_slots.p,
                                                      row_nzb.p, x, freem.p, y, dotv, parts, dflag.p); ++g_launches;
      CKL();
    });
    if (parts) gsum(parts, spmv_blocks);
  }

  template <int FF>
  int cg_solve(const double* b, double* x) {
    const int N = g.N;
    const int max_it = opt.krylov_max_iter > 0 ? opt.krylov_max_iter : std::min(20000, std::max(100, 10 * ndg()));
    const double rtol2 = cur_rtol * cur_rtol;
    CK(cudaMemsetAsync(dflag.p, 0, sizeof(int), s));
    {
      Prof::Scope ps(&prof, kcKrylov);
      k_cg_init<FF><<<kRedBlocks, kThreads, 0, s>>>(N, act_idx.p, dinv.p, b, x, kr.p, kz.p, kp.p, partials.p); ++g_launches;
      CKL();
      gsum(partials.p, 2 * kRedBlocks);
      k_finalize_sum<2><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
      CKL();
      k_cg_start<<<1, 1, 0, s>>>(sums.p, sc.p, rtol2); ++g_launches;
      CKL();
    }
    // b == 0 -> x = 0
    CK(cudaMemcpyAsync(h_sc, sc.p, sizeof(double) * kNSlots, cudaMemcpyDeviceToHost, s));
    sync();
    if (h_sc[kDone] != 0.0) return 0;
    const int batch = ndg() < 20000 ? 16 : 4;
    int done = 0;
    double* partA = partials.p;
    double* partB = partials.p + spmv_blocks;
    for (int it = 0; !done;) {
      for (int i = 0; i < batch; ++i, ++it) {
        const int par = it & 1;
        spmv(kp.p, kq.p, kp.p, partA);
        Prof::Scope ps(&prof, kcKrylov);
        k_cg_update2<FF><<<kRedBlocks, kThreads, 0, s>>>(N, act_idx.p, dinv.p, sc.p, dflag.p, par, partA, spmv_blocks,
                                                         x, kr.p, kz.p, kp.p, kq.p, partB); ++g_launches;
        gsum(partB, 2 * kRedBlocks);
        k_cg_p2<FF><<<kRedBlocks, kThreads, 0, s>>>(N, act_idx.p, sc.p, dflag.p, par, it, partB, kRedBlocks, rtol2,
                                                    max_it, kz.p, kp.p); ++g_launches;
        CKL();
      }
      CK(cudaMemcpyAsync(&done, dflag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(h_sc, sc.p, sizeof(double) * kNSlots, cudaMemcpyDeviceToHost, s));
      sync();
      prof.flush();
    }
    const int iters = static_cast<int>(h_sc[kIters]);
    if (done == 2) return -iters - 1;  // not SPD: caller falls back to BiCGStab
    if (done == 3) throw SimError(IMPM_ERR_LINEAR_SOLVER, "Krylov breakdown: NaN residual");
    if (done == 4) {
      const double rel = std::sqrt(h_sc[kRr] / h_sc[kBb]);
      if (!(rel <= 1e-6))
        throw SimError(IMPM_ERR_LINEAR_SOLVER, "CG did not converge: relative residual " + std::to_string(rel));
    }
    return iters;
  }

  // host-scalar BiCGStab (right block-Jacobi preconditioning), nonsymmetric path
  double dot(const double* a, const double* b) {
    k_dot2<<<kRedBlocks, kThreads, 0, s>>>(NF(), a, b, nullptr, nullptr, partials.p); ++g_launches;
    gsum(partials.p, 2 * kRedBlocks);
    k_finalize_sum<2><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
    CKL();
    double h[2];
    CK(cudaMemcpyAsync(h, sums.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    sync();
    return h[0];
  }
  void axpbypcz(double a, const double* x, double b, double* y, double c = 0.0, const double* z = nullptr) {
    k_axpbypcz<<<kRedBlocks, kThreads, 0, s>>>(NF(), a, x, b, y, c, z); ++g_launches;
    CKL();
  }
  template <int FF>
  void precond(const double* rin, double* z) {
    k_precond<FF><<<blocks_for(g.N), kThreads, 0, s>>>(g.N, act_idx.p, dinv.p, rin, z); ++g_launches;
    CKL();
  }
  // z = M^-1 v: MG V-cycle or block Jacobi
  template <int DD, int FE>
  const double* apply_precond(bool mgp, const double* v, double* z) {
    if (mgp) {
      vcycle<DD, FE>(0, v);
      CK(cudaMemcpyAsync(z, mg[0]->x, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
      return z;
    }
    precond<FE>(v, z);
    return z;
  }

  template <int DD, int FE>
  int bicgstab_solve(const double* b, double* x, bool mgp) {
    if (mgp) mg_setup<DD, FE>();
    CK(cudaMemsetAsync(dflag.p, 0, sizeof(int), s));
    // the u-p saddle point (cond ~1e15) needs far more than n iterations
    const int max_it = opt.krylov_max_iter > 0 ? opt.krylov_max_iter
                       : coupled              ? std::max(4000, 50 * ndg())
                                              : std::min(20000, std::max(100, 10 * ndg()));
    CK(cudaMemsetAsync(x, 0, sizeof(double) * NF(), s));
    CK(cudaMemcpyAsync(kr.p, b, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(khat.p, b, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(kp.p, 0, sizeof(double) * NF(), s));
    CK(cudaMemsetAsync(kv.p, 0, sizeof(double) * NF(), s));
    const double bb = dot(b, b);
    if (bb == 0.0) return 0;
    const double tol2 = cur_rtol * cur_rtol * bb;
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    for (int it = 1; it <= max_it; ++it) {
      const double rho_new = dot(khat.p, kr.p);
      if (rho_new == 0.0) throw SimError(IMPM_ERR_LINEAR_SOLVER, "BiCGStab breakdown (rho = 0)");
      const double beta = (rho_new / rho) * (alpha / omega);
      // p = r + beta (p - omega v)
      axpbypcz(1.0, kr.p, beta, kp.p, -beta * omega, kv.p);
      apply_precond<DD, FE>(mgp, kp.p, kz.p);  // phat in kz
      spmv(kz.p, kv.p, nullptr, nullptr);
      const double rv = dot(khat.p, kv.p);
      alpha = rho_new / rv;
      // s = r - alpha v
      CK(cudaMemcpyAsync(ks.p, kr.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
      axpbypcz(-alpha, kv.p, 1.0, ks.p);
      axpbypcz(alpha, kz.p, 1.0, x);  // x += alpha phat
      const double ss = dot(ks.p, ks.p);
      if (ss <= tol2) return it;
      apply_precond<DD, FE>(mgp, ks.p, tmp1.p);  // shat
      spmv(tmp1.p, kt.p, nullptr, nullptr);
      const double ts = dot(kt.p, ks.p), tt = dot(kt.p, kt.p);
      omega = ts / tt;
      axpbypcz(omega, tmp1.p, 1.0, x);
      // r = s - omega t
      CK(cudaMemcpyAsync(kr.p, ks.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
      axpbypcz(-omega, kt.p, 1.0, kr.p);
      const double rr = dot(kr.p, kr.p);
      if (rr <= tol2) return it;
      if (!(rr == rr)) throw SimError(IMPM_ERR_LINEAR_SOLVER, "BiCGStab breakdown: NaN residual");
      rho = rho_new;
    }
    throw SimError(IMPM_ERR_LINEAR_SOLVER, "BiCGStab did not converge");
  }


  // ------------------------------------------------ multigrid (K7 precond)
  template <int DD, int FE, int MODE>
  void level_spmv(MgLevel& L, const double* x, double* y, const double* b, double omega, const double* dotv,
                  double* parts) {
    constexpr int W = 4;
    // rows go out in 64-row chunks: small coarse levels need few CTAs (a
    // caller asking for dot partials keeps the full, fixed-size grid)
    // rows per warp: 16 on big levels (L1 reuse of x), fewer on small ones so
    // that all 148 x 32 warps get work instead of a few walking long chunks
    const int rpw = std::max(1, std::min(16, (L.n_act + spmv_blocks * W - 1) / (spmv_blocks * W)));
    const unsigned grid = parts ? spmv_blocks
                                : static_cast<unsigned>(std::max(1, std::min(mg_blocks, (L.n_act + rpw * W - 1) / (rpw * W))));
    // big levels: half-warp rows (two fp32 rows in flight per warp); the
    // denser, smaller coarse levels keep a full warp per row
    if (L.vals16)
      k_spmv<DD, FE, W, MODE, __half, 0, true><<<grid, W * 32, 0, s>>>(
          L.g, L.act_list, L.n_act, L.vals16, L.row_len16, L.row_slots, L.row_nzb, x, L.freem, y, dotv, parts, dflag.p,
          b, L.dinv, omega, rpw, mg_x4 ? L.twin(x) : nullptr, mg_x4 && MODE == kSpmvJacobi ? L.twin(y) : nullptr,
          L.rscale);
    else if (mg_f32 && L.n_act >= 50000)
      k_spmv<DD, FE, W, MODE, float, 0, true><<<grid, W * 32, 0, s>>>(
          L.g, L.act_list, L.n_act, L.vals32, L.row_len32, L.row_slots, L.row_nzb, x, L.freem, y, dotv, parts, dflag.p,
          b, L.dinv, omega, rpw, mg_x4 ? L.twin(x) : nullptr, mg_x4 && MODE == kSpmvJacobi ? L.twin(y) : nullptr);
    else if (mg_f32)
      k_spmv<DD, FE, W, MODE, float, 0><<<grid, W * 32, 0, s>>>(L.g, L.act_list, L.n_act, L.vals32, L.row_len32,
                                                                   L.row_slots, L.row_nzb, x, L.freem, y, dotv, parts,
                                                                   dflag.p, b, L.dinv, omega, rpw,
                                                                   mg_x4 ? L.twin(x) : nullptr,
                                                                   mg_x4 && MODE == kSpmvJacobi ? L.twin(y) : nullptr);
    else
      k_spmv<DD, FE, W, MODE, double, 0><<<grid, W * 32, 0, s>>>(L.g, L.act_list, L.n_act, L.vals, L.row_len, L.row_slots,
                                                            L.row_nzb, x, L.freem, y, dotv, parts, dflag.p, b, L.dinv,
                                                            omega, rpw);
    ++g_launches;
    CKL();
  }

  template <int DD, int FE>
  void mg_setup() {
    constexpr int S = ipow_c(5, DD);
    constexpr int FF = FE * FE;
    // coarse levels of an earlier load step (mg_refresh > 1): the fine level
    // is re-pointed at the current J and row structure; the stale Galerkin
    // levels stay a fixed SPD preconditioner (R = P^T under the same masks)
    // Only the CG path reuses across load steps: it alone caps the solve on
    // stale levels and rebuilds on failure (cg_mg_solve); GMRES / BiCGStab
    // always build the hierarchy of the current step.
    const bool cross_step = mg_cross_ok && mg_reuse && mg_refresh > 1 && !slab && !coupled &&
                            mg_setup_step >= 0 && mg_setup_step != step_counter &&
                            step_counter - mg_setup_step < mg_refresh && !mg.empty();
    if (cross_step) {
      MgLevel& L0 = *mg[0];
      // the fine row set changed since the levels were built: clear every
      // level-0 vector so that k_restrict (which reads the fine residual at
      // every grid node) sees zeros at nodes outside the current active set;
      // otherwise stale entries make the V-cycle affine and break PCG
      {
        const int64_t n0 = static_cast<int64_t>(L0.g.N) * FE;
        for (auto* v : {&L0.xa, &L0.xb, &L0.r, &L0.bvec}) CK(cudaMemsetAsync(v->p, 0, sizeof(double) * n0, s));
        if (FE <= 4) {
          CK(cudaMemsetAsync(L0.x4a.p, 0, sizeof(float) * L0.g.N * 4, s));
          CK(cudaMemsetAsync(L0.x4b.p, 0, sizeof(float) * L0.g.N * 4, s));
        }
        L0.x = L0.xa.p;
        L0.t = L0.xb.p;
      }
      L0.n_act = n_act;
      L0.row_len = row_len;
      L0.act_idx = act_idx.p;
      L0.act_list = act_list.p;
      L0.row_nzb = row_nzb.p;
      L0.freem = freem.p;
      L0.row_slots = row_slots.p;
      L0.vals = vals.p;
      L0.dinv = dinv.p;
      if (mg_f16) {
        vals16.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * L0.row_len16));
        rscale16.ensure(std::max(1, n_act));
        L0.vals16 = vals16.p;
        L0.rscale = rscale16.p;
      } else if (mg_f32) {
        vals32.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * L0.row_len32));
        L0.vals32 = vals32.p;
      }
    }
    if (mg_reuse && !mg.empty() &&
        (cross_step || (mg_setup_step == step_counter && mg[0]->n_act == n_act && mg[0]->vals == vals.p))) {
      if (mg_f16 && !coupled && n_act > 0) {  // fine level: fp16 smoother copy of the current J
        if (!f16_ready) {
          k_vals_to_f16<FE><<<kSpmvBlocks, 128, 0, s>>>(n_act, row_nzb.p, vals.p, row_len, vals16.p,
                                                          mg[0]->row_len16, rscale16.p);
          ++g_launches;
          CKL();
        }
      } else if (mg_f32 && n_act > 0) {  // fine level: fp32 copy of the current J
        k_vals_to_f32<FE><<<kSpmvBlocks, 128, 0, s>>>(n_act, row_nzb.p, vals.p, row_len, vals32.p, mg[0]->row_len32,
                                                        mg_f16sim);
        ++g_launches;
        CKL();
      }
      return;
    }
    mg_setup_step = step_counter;
    // level objects (and their device buffers) persist across setups; only
    // growth reallocates
    std::vector<std::unique_ptr<MgLevel>> pool;
    pool.swap(mg);
    auto take = [&pool]() {
      if (pool.empty()) return std::make_unique<MgLevel>();
      auto p = std::move(pool.front());
      pool.erase(pool.begin());
      return p;
    };
    auto L0 = take();
    L0->g = g;
    L0->n_act = n_act;
    L0->row_len = row_len;
    L0->act_idx = act_idx.p;
    L0->act_list = act_list.p;
    L0->row_nzb = row_nzb.p;
    L0->freem = freem.p;
    L0->row_slots = row_slots.p;
    L0->vals = vals.p;
    L0->dinv = dinv.p;
    L0->vals16 = nullptr;
    L0->rscale = nullptr;
    // fp16 only for the single-field solid: a u-p node row mixes the momentum
    // and mass equations, 1e10 apart, which one row scale cannot hold
    if (mg_f16 && !coupled) {
      L0->row_len16 = row_len_of<__half>(S, FE);
      vals16.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * L0->row_len16));
      rscale16.ensure(std::max(1, n_act));
      L0->vals16 = vals16.p;
      L0->rscale = rscale16.p;
      if (n_act > 0 && !f16_ready) {
        k_vals_to_f16<FE><<<kSpmvBlocks, 128, 0, s>>>(n_act, row_nzb.p, vals.p, row_len, vals16.p, L0->row_len16,
                                                        rscale16.p);
        ++g_launches;
        CKL();
      }
    } else if (mg_f32) {
      L0->row_len32 = row_len_of<float>(S, FE);
      vals32.ensure(std::max<int64_t>(1, static_cast<int64_t>(n_act) * L0->row_len32));
      L0->vals32 = vals32.p;
      if (n_act > 0) {
        k_vals_to_f32<FE><<<kSpmvBlocks, 128, 0, s>>>(n_act, row_nzb.p, vals.p, row_len, vals32.p, L0->row_len32,
                                                        mg_f16sim);
        ++g_launches;
        CKL();
      }
    }
    mg.push_back(std::move(L0));
    mg_stored_blocks = 0;
    const int coarsest_max = 200;  // unknowns solved densely at the bottom
    mg_nzb.ensure(1);
    while (static_cast<int64_t>(mg.back()->n_act) * FE > coarsest_max && mg.size() < 16) {
      MgLevel& F0 = *mg.back();
      auto C = take();
      GridC gc{};
      int N = 1;
      for (int a = 0; a < 3; ++a) {
        gc.nodes[a] = a < DD ? F0.g.nodes[a] / 2 + 1 : 1;
        gc.origin[a] = F0.g.origin[a];
        N *= gc.nodes[a];
      }
      gc.stride[DD - 1] = 1;
      for (int a = DD - 2; a >= 0; --a) gc.stride[a] = gc.stride[a + 1] * gc.nodes[a + 1];
      for (int a = DD; a < 3; ++a) gc.stride[a] = 0;
      gc.h = F0.g.h * 2.0;
      gc.N = N;
      if (N >= F0.g.N) break;  // no further coarsening possible
      C->g = gc;
      C->act_flag_b.ensure(N);
      C->act_scan_b.ensure(N + 1);
      C->act_idx_b.ensure(N);
      C->act_list_b.ensure(N);
      k_coarse_active<DD><<<blocks_for(N), kThreads, 0, s>>>(F0.g, gc, F0.act_idx, C->act_flag_b.p); ++g_launches;
      CKL();
      brick_rows<DD>(gc, C->act_flag_b.p, C->act_idx_b.p, C->act_list_b.p, C->act_scan_b.p + N);
      int na = 0;
      CK(cudaMemcpyAsync(&na, C->act_scan_b.p + N, sizeof(int), cudaMemcpyDeviceToHost, s));
      sync();
      C->n_act = na;
      C->row_len = row_len_for(S, FE);
      C->vals_b.ensure(std::max<int64_t>(1, static_cast<int64_t>(na) * C->row_len));
      C->row_slots_b.ensure(std::max<int64_t>(1, static_cast<int64_t>(na) * S));
      C->row_nzb_b.ensure(std::max(1, na));
      C->dinv_b.ensure(std::max<int64_t>(1, static_cast<int64_t>(na) * FF));
      C->freem_b.ensure(static_cast<int64_t>(N) * FE);
      CK(cudaMemsetAsync(C->freem_b.p, 0, static_cast<int64_t>(N) * FE, s));
      C->act_idx = C->act_idx_b.p;
      C->act_list = C->act_list_b.p;
      C->row_nzb = C->row_nzb_b.p;
      C->freem = C->freem_b.p;
      C->row_slots = C->row_slots_b.p;
      C->vals = C->vals_b.p;
      C->dinv = C->dinv_b.p;
      CK(cudaMemsetAsync(mg_nzb.p, 0, sizeof(unsigned long long), s));
      {
        Prof::Scope psg(&prof, kcGalerkin);
        constexpr int NT = ipow_c(4, DD);
        mg_T.ensure(std::max<int64_t>(1, static_cast<int64_t>(F0.n_act) * NT * FF));
        constexpr int W = 8;
        if (F0.n_act > 0) {
          k_galerkin_ap<DD, FE, W><<<std::min<unsigned>(blocks_for(F0.n_act, W), 148 * 8), W * 32, 0, s>>>(
              F0.g, gc, F0.n_act, F0.act_list, F0.vals, F0.row_len, F0.row_slots, F0.row_nzb, F0.freem, mg_T.p);
          ++g_launches;
          CKL();
        }
        if (na > 0) {
          k_galerkin_ptap<DD, FE, W><<<std::min<unsigned>(blocks_for(na, W), 148 * 8), W * 32, 0, s>>>(
              F0.g, gc, F0.act_idx, F0.freem, mg_T.p, C->act_list, na, C->vals_b.p, C->row_len, C->row_slots_b.p,
              C->row_nzb_b.p, C->freem_b.p, C->dinv_b.p, mg_nzb.p);
          ++g_launches;
          CKL();
        }
        if (mg_f32) {
          C->row_len32 = row_len_of<float>(S, FE);
          C->vals32_b.ensure(std::max<int64_t>(1, static_cast<int64_t>(na) * C->row_len32));
          C->vals32 = C->vals32_b.p;
          C->vals16 = nullptr;
          C->rscale = nullptr;
          if (mg_f16 && !coupled && na >= 50000) {  // big coarse level: fp16 smoother copy too
            C->row_len16 = row_len_of<__half>(S, FE);
            C->vals16_b.ensure(static_cast<int64_t>(na) * C->row_len16);
            C->rscale_b.ensure(na);
            C->vals16 = C->vals16_b.p;
            C->rscale = C->rscale_b.p;
            k_vals_to_f16<FE><<<kSpmvBlocks, 128, 0, s>>>(na, C->row_nzb_b.p, C->vals_b.p, C->row_len, C->vals16_b.p,
                                                          C->row_len16, C->rscale_b.p);
            ++g_launches;
            CKL();
          } else if (na > 0) {
            k_vals_to_f32<FE><<<kSpmvBlocks, 128, 0, s>>>(na, C->row_nzb_b.p, C->vals_b.p, C->row_len,
                                                          C->vals32_b.p, C->row_len32);
            ++g_launches;
            CKL();
          }
        }
      }
      mg.push_back(std::move(C));
    }
    // level vectors (zero outside active rows / free components)
    for (auto& Lp : mg) {
      MgLevel& L = *Lp;
      const int64_t n = static_cast<int64_t>(L.g.N) * FE;
      L.xa.ensure(n);
      L.xb.ensure(n);
      L.r.ensure(n);
      L.bvec.ensure(n);
      for (auto* v : {&L.xa, &L.xb, &L.r, &L.bvec}) CK(cudaMemsetAsync(v->p, 0, sizeof(double) * n, s));
      if (FE <= 4) {
        const int64_t n4 = static_cast<int64_t>(L.g.N) * 4;
        L.x4a.ensure(n4);
        L.x4b.ensure(n4);
        CK(cudaMemsetAsync(L.x4a.p, 0, sizeof(float) * n4, s));
        CK(cudaMemsetAsync(L.x4b.p, 0, sizeof(float) * n4, s));
      }
      L.x = L.xa.p;
      L.t = L.xb.p;
    }
    // damping of the block-Jacobi smoother from a power estimate of
    // lambda_max(Dinv A): omega = 4 / (3 lambda) (Chebyshev-optimal
    // smoothing); device-resident, one host read for all levels
    CK(cudaMemsetAsync(dflag.p, 0, sizeof(int), s));
    // lambda_max(Dinv A) moves little between the Newton iterations of one
    // load step: estimate it on the first setup of the step, then reuse
    // ... and it moves little between load steps too: omega * lambda_est =
    // 4 / 3 leaves a margin below the divergence limit 2, so the
    // estimate is refreshed every 5 load steps (or when the depth changes)
    const bool need_power =
        mg_power_step < 0 || step_counter - mg_power_step >= mg_power_every || mg_lam_host.size() != mg.size();
    mg_lam.ensure(std::max<size_t>(mg.size(), 1));
    if (need_power) {
      Prof::Scope psp(&prof, kcMgPower);
      for (size_t l = 0; l + 1 < mg.size(); ++l) {
        MgLevel& L = *mg[l];
        const int64_t n = static_cast<int64_t>(L.g.N) * FE;
        k_fill_free<<<blocks_for(n), kThreads, 0, s>>>(n, L.freem, L.bvec.p); ++g_launches;
        CKL();
        for (int it = 0; it < 8; ++it) {
          level_spmv<DD, FE, kSpmvY>(L, L.bvec.p, L.r.p, nullptr, 0.0, nullptr, nullptr);
          k_precond<FE><<<blocks_for(L.g.N), kThreads, 0, s>>>(L.g.N, L.act_idx, L.dinv, L.r.p, L.t); ++g_launches;
          k_dot2<<<kRedBlocks, kThreads, 0, s>>>(n, L.t, L.t, L.bvec.p, L.bvec.p, partials.p); ++g_launches;
          k_finalize_sum<2><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
          k_power_step<<<kRedBlocks, kThreads, 0, s>>>(n, sums.p, L.t, L.bvec.p, mg_lam.p + l); ++g_launches;
          CKL();
        }
      }
    }
    {
      std::vector<double> lam(mg.size(), 1.0);
      if (need_power) {
        if (mg.size() > 1)
          CK(cudaMemcpyAsync(lam.data(), mg_lam.p, sizeof(double) * (mg.size() - 1), cudaMemcpyDeviceToHost, s));
        sync();
        mg_lam_host = lam;
        mg_power_step = step_counter;
      } else {
        lam = mg_lam_host;
      }
      for (size_t l = 0; l + 1 < mg.size(); ++l) {
        MgLevel& L = *mg[l];
        const int64_t n = static_cast<int64_t>(L.g.N) * FE;
        const double sf = l > 0 && mg_omega_safety_coarse > 0.0 ? mg_omega_safety_coarse : mg_omega_safety;
        L.omega = 4.0 / (3.0 * sf * (lam[l] > 0 ? lam[l] : 1.0));
        CK(cudaMemsetAsync(L.t, 0, sizeof(double) * n, s));
        CK(cudaMemsetAsync(L.bvec.p, 0, sizeof(double) * n, s));
        CK(cudaMemsetAsync(L.r.p, 0, sizeof(double) * n, s));
      }
    }
    Prof::Scope psc(&prof, kcMgCoarsest);
    // coarsest: dense inverse over (active row, component), identity on non-free
    MgLevel& B = *mg.back();
    const int nb = B.n_act, n = nb * FE;
    mg_dense_n = n;
    if (n > 0) {
      std::vector<int> slots_nzb(nb);
      std::vector<uint8_t> slots(static_cast<size_t>(nb) * S), fm(static_cast<size_t>(B.g.N) * FE);
      std::vector<int> alist(nb), aidx(B.g.N);
      std::vector<double> vals_h(static_cast<size_t>(nb) * B.row_len), dense(static_cast<size_t>(n) * n, 0.0);
      CK(cudaMemcpyAsync(slots_nzb.data(), B.row_nzb, sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(slots.data(), B.row_slots, slots.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(fm.data(), B.freem, fm.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(alist.data(), B.act_list, sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(aidx.data(), B.act_idx, sizeof(int) * B.g.N, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(vals_h.data(), B.vals, sizeof(double) * vals_h.size(), cudaMemcpyDeviceToHost, s));
      sync();
      for (int rrow = 0; rrow < nb; ++rrow) {
        const int k = alist[rrow];
        int kidx[3] = {0, 0, 0};
        for (int a = 0; a < DD; ++a) kidx[a] = (k / B.g.stride[a]) % B.g.nodes[a];
        for (int pos = 0; pos < slots_nzb[rrow]; ++pos) {
          int sl = slots[static_cast<size_t>(rrow) * S + pos], nbn = 0;
          int rel[3];
          for (int a = DD - 1; a >= 0; --a) {
            rel[a] = sl % 5 - 2;
            sl /= 5;
          }
          bool ok = true;
          for (int a = 0; a < DD; ++a) {
            const int ia = kidx[a] + rel[a];
            ok = ok && ia >= 0 && ia < B.g.nodes[a];
            nbn += ia * B.g.stride[a];
          }
          if (!ok) continue;
          const int crow = aidx[nbn];
          if (crow < 0) continue;
          for (int c = 0; c < FE; ++c)
            for (int d = 0; d < FE; ++d)
              if (fm[static_cast<size_t>(k) * FE + c] && fm[static_cast<size_t>(nbn) * FE + d])
                dense[static_cast<size_t>(rrow * FE + c) * n + crow * FE + d] =
                    vals_h[static_cast<size_t>(rrow) * B.row_len + c * cpad(slots_nzb[rrow], FE) + pos * FE + d];
        }
        for (int c = 0; c < FE; ++c)
          if (!fm[static_cast<size_t>(k) * FE + c]) dense[static_cast<size_t>(rrow * FE + c) * n + rrow * FE + c] = 1.0;
      }
      std::vector<double> inv = invert_dense(dense, n);
      mg_dense.ensure(static_cast<size_t>(n) * n);
      CK(cudaMemcpyAsync(mg_dense.p, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice, s));
      sync();
    }
  }

  // Gauss-Jordan with partial pivoting (coarsest level, n <= ~600)
  static std::vector<double> invert_dense(std::vector<double> a, int n) {
    std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + i] = 1.0;
    for (int c = 0; c < n; ++c) {
      int p = c;
      for (int r2 = c + 1; r2 < n; ++r2)
        if (std::abs(a[static_cast<size_t>(r2) * n + c]) > std::abs(a[static_cast<size_t>(p) * n + c])) p = r2;
      if (a[static_cast<size_t>(p) * n + c] == 0.0) continue;  // singular direction: leave it
      if (p != c)
        for (int j = 0; j < n; ++j) {
          std::swap(a[static_cast<size_t>(p) * n + j], a[static_cast<size_t>(c) * n + j]);
          std::swap(inv[static_cast<size_t>(p) * n + j], inv[static_cast<size_t>(c) * n + j]);
        }
      const double d = 1.0 / a[static_cast<size_t>(c) * n + c];
      for (int j = 0; j < n; ++j) {
        a[static_cast<size_t>(c) * n + j] *= d;
        inv[static_cast<size_t>(c) * n + j] *= d;
      }
      for (int r2 = 0; r2 < n; ++r2) {
        if (r2 == c) continue;
        const double f = a[static_cast<size_t>(r2) * n + c];
        if (f == 0.0) continue;
        for (int j = 0; j < n; ++j) {
          a[static_cast<size_t>(r2) * n + j] -= f * a[static_cast<size_t>(c) * n + j];
          inv[static_cast<size_t>(r2) * n + j] -= f * inv[static_cast<size_t>(c) * n + j];
        }
      }
    }
    return inv;
  }

  // z = V-cycle(b) at level l; result in mg[l]->x
  template <int DD, int FE>
  void vcycle(size_t l, const double* b) {
    MgLevel& L = *mg[l];
    const int lcls = l == 0 ? kcVcL0 : (l == 1 ? kcVcL1 : kcVcCoarse);  // nested sub-classes of "vcycle"
    if (l + 1 == mg.size()) {
      if (mg_dense_n > 0) {
        Prof::Scope ps(&prof, kcVcCoarse);
        k_dense_apply<<<std::min<unsigned>(blocks_for(mg_dense_n, 128), 148), 128, 0, s>>>(
            mg_dense_n, FE, dflag.p, L.act_list, mg_dense.p, b, L.x); ++g_launches;
        CKL();
      }
      return;
    }
    const int nu0 = mg_smooth_env > 0 ? mg_smooth_env : (opt.mg_smooth > 0 ? opt.mg_smooth : 1);
    const int nu = l > 0 && mg_nu_coarse > 0 ? mg_nu_coarse : nu0;
    MgLevel& C = *mg[l + 1];
    {
      Prof::Scope ps(&prof, lcls);
      // pre-smoothing from x = 0
      k_jacobi0<FE><<<kRedBlocks, kThreads, 0, s>>>(L.n_act, dflag.p, L.act_list, L.dinv, L.freem, L.omega, b, L.x,
                                                    mg_x4 ? L.twin(L.x) : nullptr);
      ++g_launches;
      CKL();
      for (int i = 1; i < nu; ++i) {
        level_spmv<DD, FE, kSpmvJacobi>(L, L.x, L.t, b, L.omega, nullptr, nullptr);
        std::swap(L.x, L.t);
      }
      level_spmv<DD, FE, kSpmvResid>(L, L.x, L.r.p, b, 0.0, nullptr, nullptr);
      k_restrict<DD, FE><<<blocks_for(C.g.N), kThreads, 0, s>>>(L.g, C.g, dflag.p, L.r.p, C.freem, C.bvec.p);
      ++g_launches;
      CKL();
    }
    vcycle<DD, FE>(l + 1, C.bvec.p);
    Prof::Scope ps(&prof, lcls);
    k_prolong_add<DD, FE><<<blocks_for(L.g.N), kThreads, 0, s>>>(L.g, C.g, dflag.p, C.x, L.freem, L.x,
                                                                  mg_x4 ? L.twin(L.x) : nullptr);
    ++g_launches;
    CKL();
    for (int i = 0; i < nu; ++i) {
      level_spmv<DD, FE, kSpmvJacobi>(L, L.x, L.t, b, L.omega, nullptr, nullptr);
      std::swap(L.x, L.t);
    }
  }


  // MG-preconditioned CG (device-resident scalars, batched host checks)
  template <int DD, int FE>
  int cg_mg_solve(const double* b, double* x) {
    // stale coarse levels (mg_refresh): try with a cap, rebuild and retry on failure
    if (mg_reuse && mg_refresh > 1 && !slab && !coupled) {
      const bool will_reuse = mg_setup_step >= 0 && mg_setup_step != step_counter &&
                              step_counter - mg_setup_step < mg_refresh && !mg.empty();
      if (will_reuse && last_cg_iters > 0) {
        int it = -1;
        mg_cross_ok = true;
        try {
          it = cg_mg_solve_once<DD, FE>(b, x, std::max(50, 4 * last_cg_iters));
        } catch (const SimError& e) {
          mg_cross_ok = false;
          if (e.code != IMPM_ERR_LINEAR_SOLVER) throw;
          it = -1;
        }
        mg_cross_ok = false;
        if (it >= 0) return last_cg_iters = it;
        mg_setup_step = -1;  // rebuild the hierarchy for the current J and retry
      }
    }
    const int it = cg_mg_solve_once<DD, FE>(b, x, 0);
    if (it >= 0) last_cg_iters = it;
    return it;
  }

  template <int DD, int FE>
  int cg_mg_solve_once(const double* b, double* x, int cap) {
    const int N = g.N;
    const int64_t n = NF();
    const int max_it = cap > 0                   ? cap
                       : opt.krylov_max_iter > 0 ? opt.krylov_max_iter
                                                 : std::min(20000, std::max(100, 10 * ndg()));
    const double rtol2 = cur_rtol * cur_rtol;
    {
      Prof::Scope ps(&prof, kcMgSetup);
      mg_setup<DD, FE>();
    }
    CK(cudaMemsetAsync(dflag.p, 0, sizeof(int), s));
    double* partA = partials.p;
    double* partB = partials.p + spmv_blocks;
    CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    CK(cudaMemcpyAsync(kr.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    {
      Prof::Scope ps(&prof, kcVcycle);
      vcycle<DD, FE>(0, kr.p);
    }
    const double* z = mg[0]->x;
    CK(cudaMemcpyAsync(kp.p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    k_dot2<<<kRedBlocks, kThreads, 0, s>>>(n, kr.p, z, b, b, partials.p); ++g_launches;
    gsum(partials.p, 2 * kRedBlocks);
    k_finalize_sum<2><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
    k_cg_start<<<1, 1, 0, s>>>(sums.p, sc.p, rtol2); ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(h_sc, sc.p, sizeof(double) * kNSlots, cudaMemcpyDeviceToHost, s));
    sync();
    if (h_sc[kDone] != 0.0) return 0;
    const int batch = ndg() < 20000 ? 8 : 4;
    int done = 0;
    for (int it = 0; !done;) {
      for (int i = 0; i < batch; ++i, ++it) {
        const int par = it & 1;
        spmv(kp.p, kq.p, kp.p, partA);
        {
          Prof::Scope ps(&prof, kcKrylov);
          k_cg_update_mg<FE><<<kRedBlocks, kThreads, 0, s>>>(N, act_idx.p, sc.p, dflag.p, par, partA, spmv_blocks, x,
                                                             kr.p, kp.p, kq.p, partB + kRedBlocks); ++g_launches;
          CKL();
        }
        {
          Prof::Scope ps(&prof, kcVcycle);
          vcycle<DD, FE>(0, kr.p);
        }
        z = mg[0]->x;
        Prof::Scope ps(&prof, kcKrylov);
        k_dot1<<<kRedBlocks, kThreads, 0, s>>>(n, dflag.p, kr.p, z, partB); ++g_launches;
        gsum(partB, 2 * kRedBlocks);
        k_cg_p2<FE><<<kRedBlocks, kThreads, 0, s>>>(N, act_idx.p, sc.p, dflag.p, par, it, partB, kRedBlocks, rtol2,
                                                    max_it, z, kp.p); ++g_launches;
        CKL();
      }
      CK(cudaMemcpyAsync(&done, dflag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(h_sc, sc.p, sizeof(double) * kNSlots, cudaMemcpyDeviceToHost, s));
      sync();
      prof.flush();
    }
    const int iters = static_cast<int>(h_sc[kIters]);
    if (done == 2) return -iters - 1;
    if (done == 3) throw SimError(IMPM_ERR_LINEAR_SOLVER, "Krylov breakdown: NaN residual");
    if (done == 4) {
      if (cap > 0) return -1;  // capped attempt on stale levels: the caller rebuilds and retries
      const double rel = std::sqrt(h_sc[kRr] / h_sc[kBb]);
      if (!(rel <= 1e-6))
        throw SimError(IMPM_ERR_LINEAR_SOLVER, "MG-CG did not converge: relative residual " + std::to_string(rel));
    }
    return iters;
  }


  // GMRES(m), right-preconditioned (block Jacobi or MG), modified
  // Gram-Schmidt on device vectors, Hessenberg/Givens on the host.
  // Robust path for the nonsymmetric, badly scaled u-p saddle point.
  DBuf<double> gm_V, gm_part, gm_h;
  static constexpr int kGmBlocks = 148;
  double dot_sync(const double* a, const double* b) {
    k_dot2<<<kRedBlocks, kThreads, 0, s>>>(NF(), a, b, nullptr, nullptr, partials.p); ++g_launches;
    gsum(partials.p, 2 * kRedBlocks);
    k_finalize_sum<2><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
    CKL();
    double hh[2];
    CK(cudaMemcpyAsync(hh, sums.p, sizeof(hh), cudaMemcpyDeviceToHost, s));
    sync();
    return hh[0];
  }

  template <int DD, int FE>
  int gmres_solve(const double* b, double* x, bool mgp) {
    const int64_t n = NF();
    const int m = std::max(2, std::min(300, ndg()));
    gm_part.ensure(static_cast<size_t>(m + 1) * kGmBlocks);
    gm_h.ensure(m + 1);
    std::vector<double> hbuf(m + 1);
    const int max_it = opt.krylov_max_iter > 0 ? opt.krylov_max_iter
                       : mgp                   ? 5000
                                               : std::min(20000, std::max(2000, 20 * ndg()));
    if (mgp) mg_setup<DD, FE>();
    CK(cudaMemsetAsync(dflag.p, 0, sizeof(int), s));
    gm_V.ensure(static_cast<size_t>(m + 1) * n);
    // SpMV / preconditioners write active rows only: the basis must start at
    // zero so inactive entries never carry stale memory into the dots
    CK(cudaMemsetAsync(gm_V.p, 0, sizeof(double) * static_cast<size_t>(m + 1) * n, s));
    CK(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    const double bnorm = std::sqrt(dot_sync(b, b));
    if (bnorm == 0.0) return 0;
    const double tol = cur_rtol * bnorm;
    std::vector<double> H(static_cast<size_t>(m + 1) * m), cs(m), sn(m), gv(m + 1), y(m);
    int total = 0;
    CK(cudaMemcpyAsync(kr.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));  // r = b (x = 0)
    double beta = bnorm, prev_beta = INFINITY;
    while (total < max_it) {
      double* V0 = gm_V.p;
      axpbypcz(1.0 / beta, kr.p, 0.0, V0);
      std::fill(gv.begin(), gv.end(), 0.0);
      gv[0] = beta;
      int j = 0;
      for (; j < m && total < max_it; ++j, ++total) {
        double* Vj = gm_V.p + static_cast<size_t>(j) * n;
        double* w = gm_V.p + static_cast<size_t>(j + 1) * n;
        apply_precond<DD, FE>(mgp, Vj, kz.p);
        spmv(kz.p, w, nullptr, nullptr);
        // classical Gram-Schmidt, twice (CGS2): batched dots on the device
        for (int i = 0; i <= j; ++i) H[static_cast<size_t>(i) * m + j] = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          k_vdot<<<dim3(kGmBlocks, j + 1), kThreads, 0, s>>>(n, gm_V.p, n, w, gm_part.p); ++g_launches;
          gsum(gm_part.p, static_cast<size_t>(j + 1) * kGmBlocks);
          k_finalize_rows<<<j + 1, 256, 0, s>>>(gm_part.p, kGmBlocks, gm_h.p); ++g_launches;
          k_vsub<<<kRedBlocks, kThreads, 0, s>>>(n, gm_V.p, n, j + 1, gm_h.p, w); ++g_launches;
          CKL();
          CK(cudaMemcpyAsync(hbuf.data(), gm_h.p, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
          sync();
          for (int i = 0; i <= j; ++i) H[static_cast<size_t>(i) * m + j] += hbuf[i];
        }
        const double hn = std::sqrt(dot_sync(w, w));
        H[static_cast<size_t>(j + 1) * m + j] = hn;
        if (hn > 0.0) axpbypcz(1.0 / hn, w, 0.0, w);
        for (int i = 0; i < j; ++i) {  // apply previous rotations
          const double a = H[static_cast<size_t>(i) * m + j], bb = H[static_cast<size_t>(i + 1) * m + j];
          H[static_cast<size_t>(i) * m + j] = cs[i] * a + sn[i] * bb;
          H[static_cast<size_t>(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
        }
        const double a = H[static_cast<size_t>(j) * m + j], bb = H[static_cast<size_t>(j + 1) * m + j];
        const double rr = std::hypot(a, bb);
        cs[j] = rr > 0 ? a / rr : 1.0;
        sn[j] = rr > 0 ? bb / rr : 0.0;
        H[static_cast<size_t>(j) * m + j] = rr;
        H[static_cast<size_t>(j + 1) * m + j] = 0.0;
        gv[j + 1] = -sn[j] * gv[j];
        gv[j] = cs[j] * gv[j];
        if (std::abs(gv[j + 1]) <= tol || hn == 0.0) {
          ++j;
          ++total;
          break;
        }
      }
      // y = H^-1 g (upper triangular j x j); u = V y; x += M^-1 u
      for (int i = j - 1; i >= 0; --i) {
        double acc = gv[i];
        for (int k2 = i + 1; k2 < j; ++k2) acc -= H[static_cast<size_t>(i) * m + k2] * y[k2];
        y[i] = H[static_cast<size_t>(i) * m + i] != 0.0 ? acc / H[static_cast<size_t>(i) * m + i] : 0.0;
      }
      CK(cudaMemsetAsync(tmp1.p, 0, sizeof(double) * n, s));
      for (int i = 0; i < j; ++i) axpbypcz(y[i], gm_V.p + static_cast<size_t>(i) * n, 1.0, tmp1.p);
      apply_precond<DD, FE>(mgp, tmp1.p, kz.p);
      axpbypcz(1.0, kz.p, 1.0, x);
      // true residual
      spmv(x, kq.p, nullptr, nullptr);
      CK(cudaMemcpyAsync(kr.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      axpbypcz(-1.0, kq.p, 1.0, kr.p);
      beta = std::sqrt(dot_sync(kr.p, kr.p));
      if (krylov_debug)
        std::fprintf(stderr, "[gmres] it %d true rel %.3e target %.3e (arnoldi est %.3e)\n", total, beta / bnorm,
                     tol / bnorm, std::abs(gv[j]) / bnorm);
      if (!(beta == beta)) throw SimError(IMPM_ERR_LINEAR_SOLVER, "GMRES breakdown: NaN residual");
      if (beta <= tol) return total;
      // attainable accuracy: the Arnoldi estimate met the target but the true
      // residual did not move over a restart (rounding in b - Jx at cond ~1e15
      // with a tiny warm-started rhs). The Newton test decides from here.
      if (std::abs(gv[j]) <= tol && beta > 0.5 * prev_beta && beta <= 1e-3 * bnorm) return total;
      prev_beta = beta;
    }
    const double rel = beta / bnorm;
    if (!(rel <= 1e-6)) throw SimError(IMPM_ERR_LINEAR_SOLVER, "GMRES did not converge: relative residual " +
                                                                   std::to_string(rel));
    return total;
  }
  // delta = J^-1 rhs (grid layout); returns Krylov iterations. Symmetric
  // single-field J: CG (MG or block-Jacobi preconditioned), falling back to
  // BiCGStab on breakdown; coupled u-p (nonsymmetric): BiCGStab.
  // Direct path (small systems): the reference's own algorithm, sparse_lu_solve
  // (src/linear_solver.cpp:11-88: row equilibration, pivoted LU, <= 2
  // refinement sweeps, backward-error gate), on the CSR of J over the free DOFs
  // (the reference pattern, jacobian.hpp:36-65), device-resident end to end.
  // Used by the auto solver for n_dofs <= kDirectMax on one GPU: below that
  // size a dense device LU costs milliseconds, and it resolves the numerically
  // singular systems of non-lattice particle sets (fringe nodes at ~1e-14 of
  // the bulk stiffness, cond(S J) ~ 1e19) exactly as the reference's LU does,
  // which no Krylov method can.
  static constexpr int kDirectMax = csr::kDenseMax;
  std::unique_ptr<csr::LuSolver> lu;
  DBuf<int32_t> lu_cols;
  DBuf<double> lu_vals, lu_b, lu_x;
  bool use_direct() const {
    return opt.krylov == IMPM_KRYLOV_AUTO && !multi() && n_dofs > 0 && n_dofs <= kDirectMax && !direct_off;
  }
  bool direct_off = std::getenv("IMPM_DIRECT") && std::atoi(std::getenv("IMPM_DIRECT")) == 0;
  int direct_solve(const double* rhs, double* x) {
    const int n = n_dofs;
    const int64_t z = ref_nnz();
    std::vector<int64_t> rl(n), rp(n + 1, 0);
    CK(cudaMemcpyAsync(rl.data(), rowlen.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    sync();
    for (int i = 0; i < n; ++i) rp[i + 1] = rp[i] + rl[i];
    CK(cudaMemcpyAsync(rowptr.p, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    lu_cols.ensure(std::max<int64_t>(z, 1));
    lu_vals.ensure(std::max<int64_t>(z, 1));
    lu_b.ensure(n);
    lu_x.ensure(n);
    dispatch_df([&](auto Dc, auto Fc) {
      constexpr int DD = decltype(Dc)::value, FE = decltype(Fc)::value;
      k_csr_fill<DD, FE><<<blocks_for(n), kThreads, 0, s>>>(g, n, node_of.p, field_of.p, dof_of.p, act_idx.p, vals.p,
                                                            row_len, row_slots.p, row_nzb.p, rowptr.p, lu_cols.p,
                                                            lu_vals.p); ++g_launches;
      CKL();
    });
    k_grid_to_dof<<<blocks_for(n), kThreads, 0, s>>>(n, rhs, node_of.p, field_of.p, F, lu_b.p); ++g_launches;
    CKL();
    if (!lu) lu = std::make_unique<csr::LuSolver>();
    lu->A.upload_device(n, rowptr.p, lu_cols.p, lu_vals.p, z, s);
    lu->solve_device(lu_b.p, lu_x.p);
    CK(cudaMemsetAsync(x, 0, sizeof(double) * NF(), s));
    k_dof_to_grid<<<blocks_for(n), kThreads, 0, s>>>(n, lu_x.p, node_of.p, field_of.p, F, x); ++g_launches;
    CKL();
    return 0;
  }

  int solve_dev(const double* rhs, double* x) {
    if (use_direct()) return direct_solve(rhs, x);
    int out = 0;
    dispatch_df([&](auto Dc, auto Fc) {
      constexpr int DD = decltype(Dc)::value, FE = decltype(Fc)::value;
      // non-associative Drucker-Prager flow gives a nonsymmetric J -> GMRES;
      // MG right-preconditions GMRES for DP; the u-p saddle point uses block Jacobi
      const bool nonsym = coupled || mat.kind == kDruckerPrager || mat.kind == kCamClay;
      // u-p: GMRES right-preconditioned by the same geometric MG on the 3x3
      // node blocks (u_x, u_y, p): the block-Jacobi smoother inverts each
      // node's u-p coupling, Galerkin coarse levels keep it
      const bool mgp = opt.precond == IMPM_PRECOND_MG;
      if (!nonsym && opt.krylov != IMPM_KRYLOV_BICGSTAB && opt.krylov != IMPM_KRYLOV_GMRES) {
        const int it = mgp ? cg_mg_solve<DD, FE>(rhs, x) : cg_solve<FE>(rhs, x);
        if (it >= 0) {
          out = it;
          return;
        }
        if (opt.krylov == IMPM_KRYLOV_CG) throw SimError(IMPM_ERR_LINEAR_SOLVER, "CG breakdown: J not SPD");
        // p.Jp <= 0: J is indefinite or numerically singular (fringe nodes
        // carrying ~1e-14 of the bulk stiffness) -> GMRES, same preconditioner
        out = -it - 1 + gmres_solve<DD, FE>(rhs, x, mgp);
        return;
      }
      if (nonsym || opt.krylov == IMPM_KRYLOV_GMRES) {
        if (!mgp) {
          out = gmres_solve<DD, FE>(rhs, x, false);
          return;
        }
        try {
          out = gmres_solve<DD, FE>(rhs, x, true);
        } catch (const SimError& e) {
          // MG smoothing can diverge on a nonsymmetric J with (near-)singular
          // node blocks (Drucker-Prager particles projected to the cone tip
          // carry no stiffness): retry with block Jacobi before giving up
          if (e.code != IMPM_ERR_LINEAR_SOLVER) throw;
          if (krylov_debug) std::fprintf(stderr, "[gmres] MG failed (%s): block-Jacobi retry\n", e.what());
          mg_setup_step = -1;  // the next MG solve rebuilds the hierarchy
          out = gmres_solve<DD, FE>(rhs, x, false);
        }
        return;
      }
      out = bicgstab_solve<DD, FE>(rhs, x, mgp);
    });
    return out;
  }

  // ------------------------------------------------------ Newton (a16/a17)
  impm_step_record* rec_ = nullptr;
  std::vector<double> rels_;

  void finish_record(impm_step_record* rec, const std::vector<double>& rels) {
    if (!rec) return;
    rec->n_rel = static_cast<int>(rels.size());
    if (rec->rel_residuals)
      for (int i = 0; i < std::min<int>(rec->n_rel, rec->rel_capacity); ++i) rec->rel_residuals[i] = rels[i];
  }

  int64_t ref_nnz_cache = -1;
  int64_t ref_nnz() {
    if (ref_nnz_cache >= 0) return ref_nnz_cache;
    rowlen.ensure(std::max(n_dofs, 1) + 1);
    rowptr.ensure(std::max(n_dofs, 1) + 1);
    if (n_dofs == 0) return ref_nnz_cache = 0;
    dispatch_df([&](auto Dc, auto Fc) {
      constexpr int DD = decltype(Dc)::value, FE = decltype(Fc)::value;
      k_csr_count<DD, FE><<<blocks_for(n_dofs), kThreads, 0, s>>>(g, n_dofs, node_of.p, dof_of.p, rowlen.p); ++g_launches;
      CKL();
    });
    // summed on the device (the host loop over 3 M row lengths and their
    // 25 MB download cost ~5 ms per load step at cfg 4); rank-local on a slab
    k_sum_i64<<<kRedBlocks, kThreads, 0, s>>>(n_dofs, rowlen.p, partials.p); ++g_launches;
    k_finalize_sum<1><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, sums.p); ++g_launches;
    CKL();
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, sums.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    sync();
    return ref_nnz_cache = std::llround(h);
  }

  // newton_attempt (mpm_solver.hpp:281-355); u already holds u_init
  // r0_known >= 0: r already holds r(u) with that norm (the warm-start test
  // of newton_solve evaluated it; mpm_solver.hpp:297 recomputes the same value)
  void newton_attempt(double load_scale, impm_step_record* rec, double r0_known = -1.0) {
    exact_newton = exact_newton_env >= 0 ? exact_newton_env != 0 : mat.kind == kHenckyJ2;
    std::vector<double> rels;
    const auto t0 = std::chrono::steady_clock::now();
    double diff_s = 0.0, solve_s = 0.0, res_s = 0.0, rnorm_prev = 0.0, ratio1_now = -1.0;
    int kry = 0, iters = 0;
    auto tres = std::chrono::steady_clock::now();
    const double r0 = r0_known >= 0.0 ? r0_known : residual_dev(u.p, load_scale, r.p);
    res_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tres).count();
    auto fill = [&]() {
      if (!rec) return;
      rec->step = step_counter;
      rec->iterations = iters;
      rec->r0_norm = r0;
      rec->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      rec->diff_seconds = diff_s;
      rec->solve_seconds = solve_s;
      rec->residual_seconds = res_s;
      rec->krylov_iterations = kry;
      // jacobian.hpp:117-125 (sparse: fields * b^D passes) or :71-91 (dense: one per dof)
      rec->backward_passes = iters * (opt.strategy == IMPM_STRATEGY_DENSE ? ndg() : F * ipow_c(5, D));
      rec->nnz_assembled = iters * ref_nnz();
      finish_record(rec, rels);
    };
    if (r0 < opt.abs_floor) {
      fill();
      return;
    }
    for (int it = 1; it <= opt.max_iterations; ++it) {
      auto tj = std::chrono::steady_clock::now();
      jacobian_dev(u.p);
      sync();
      diff_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tj).count();
      // rhs = -r. Inexact Newton with a count-preserving forcing term: the
      // linear residual |J d + r| <= eta |r| with eta = 0.01 tol r0 / |r|
      // adds at most 1% of tol * r0 to the next Newton residual, so the
      // convergence test (mpm_solver.hpp:334-337) sees the exact-solve
      // outcome; floor = krylov_rtol (1e-12).
      auto ts = std::chrono::steady_clock::now();
      axpbypcz(-1.0, r.p, 0.0, tmp2.p);
      if (exact_newton) {
        // return-map materials: the elastic/plastic branch of every particle
        // (materials.hpp:185-190) is decided on the iterate, so an inexact
        // step can flip a branch the reference's LU (backward error ~1e-14,
        // linear_solver.cpp:71-78) does not; solve to the exact-solve target
        cur_rtol = exact_rtol;
      } else if (it == 1) {
        // first iteration: its linear error lands in r1 as <= eta r0, so eta =
        // 1% of the contraction |r1| / r0 seen at the previous load step keeps
        // r1 within ~1% of the exact-solve value (no history: 1% of tol)
        const double ref = newton_ratio1 > 0.0 ? std::max(newton_ratio1, opt.tol) : opt.tol;
        cur_rtol = std::min(1e-6, std::max(opt.krylov_rtol, newton_eta_factor * ref));
      } else {
        cur_rtol = std::min(1e-6, std::max(opt.krylov_rtol, 0.01 * opt.tol * r0 / std::max(rnorm_prev, 1e-300)));
      }
      kry += solve_dev(tmp2.p, delta.p);
      cur_rtol = opt.krylov_rtol;
      solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
      // full step; backtrack only while infeasible (mpm_solver.hpp:313-332)
      double alpha = 1.0, rnorm = 0.0;
      bool accepted = false;
      for (int cut = 0; cut < 12 && !accepted; ++cut, alpha *= 0.5) {
        CK(cudaMemcpyAsync(utry.p, u.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
        axpbypcz(alpha, delta.p, 1.0, utry.p);
        try {
          tres = std::chrono::steady_clock::now();
          rnorm = residual_dev(utry.p, load_scale, rtry.p);
          res_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tres).count();
          std::swap(u.p, utry.p);
          std::swap(r.p, rtry.p);
          rnorm_prev = rnorm;
          accepted = true;
          if (it == 1) ratio1_now = rnorm / r0;
        } catch (const SimError& e) {
          if (e.code != IMPM_ERR_DOMAIN) throw;
        }
      }
      if (!accepted) {
        fill();
        throw SimError(IMPM_ERR_NONCONVERGENCE, "Newton stalled at step " + std::to_string(step_counter), rels);
      }
      const double rel = rnorm / r0;
      rels.push_back(rel);
      iters = it;
      if (rel <= opt.tol) {
        newton_ratio1 = ratio1_now;
        if (opt.total_lagrangian) {
          have_uwarm = true;
          CK(cudaMemcpyAsync(prev.p, u.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
        } else {
          have_prev = true;
          CK(cudaMemcpyAsync(prev.p, u.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
        }
        sync();
        fill();
        return;
      }
    }
    fill();
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", opt.tol);
    throw SimError(IMPM_ERR_NONCONVERGENCE,
                   std::string("Newton did not reach tol ") + buf + " in " + std::to_string(opt.max_iterations) +
                       " iterations at step " + std::to_string(step_counter),
                   rels);
  }

  // newton_solve (mpm_solver.hpp:248-279)
  void newton_solve(double load_scale, impm_step_record* rec) {
    if (!step_built) throw SimError(IMPM_ERR_CONFIG, "newton_solve before begin_step");
    ref_nnz_cache = -1;
    const bool have_warm = opt.total_lagrangian ? have_uwarm : have_prev;
    ++step_counter;
    if (have_warm) {
      // warm = previous converged solution restricted to the current free DOFs
      mask_copy(prev.p, tmp1.p);
      bool warm_viable = true;
      double r_warm = 0.0;
      try {
        r_warm = residual_dev(tmp1.p, load_scale, r.p);
      } catch (const SimError& e) {
        if (e.code != IMPM_ERR_DOMAIN) throw;
        warm_viable = false;
      }
      if (warm_viable) {
        CK(cudaMemsetAsync(utry.p, 0, sizeof(double) * NF(), s));
        const double r_cold = residual_dev(utry.p, load_scale, rtry.p);
        if (r_warm < r_cold) {
          CK(cudaMemcpyAsync(u.p, tmp1.p, sizeof(double) * NF(), cudaMemcpyDeviceToDevice, s));
          try {
            newton_attempt(load_scale, rec, r_warm);  // r holds r(u_warm)
            return;
          } catch (const SimError& e) {
            if (e.code != IMPM_ERR_NONCONVERGENCE) throw;
          }
        } else {  // cold start: rtry holds r(0)
          CK(cudaMemsetAsync(u.p, 0, sizeof(double) * NF(), s));
          std::swap(r.p, rtry.p);
          newton_attempt(load_scale, rec, r_cold);
          return;
        }
      }
    }
    CK(cudaMemsetAsync(u.p, 0, sizeof(double) * NF(), s));
    newton_attempt(load_scale, rec);
  }

  // dst = src at free DOFs, 0 elsewhere (grid layout)
  void mask_copy(const double* src, double* dst) {
    // via dof vectors: dst = 0; dst[node_of,field_of] = src[...]
    CK(cudaMemsetAsync(dst, 0, sizeof(double) * NF(), s));
    if (n_dofs == 0) return;
    tmp2.ensure(NF());
    k_grid_to_dof<<<blocks_for(n_dofs), kThreads, 0, s>>>(n_dofs, src, node_of.p, field_of.p, F, kt.p); ++g_launches;
    k_dof_to_grid<<<blocks_for(n_dofs), kThreads, 0, s>>>(n_dofs, kt.p, node_of.p, field_of.p, F, dst); ++g_launches;
    CKL();
  }


  // ------------------------------- coupled u-p (2D reference F=3; 3D extension F=4)
  PoroC poro_c() const {
    PoroC q = pc;
    q.g0 = gravity[0];
    q.g1 = gravity[1];
    q.g2 = gravity[2];
    return q;
  }

  // CoupledSim::assemble<double> (porous.hpp:127-186); dt > 0 required
  template <class Fn>
  void dispatch_up(Fn&& fn) {  // (D, shape) of a coupled simulation
    if (D == 2) {
      if (shape == 2) fn(IC<2>{}, IC<2>{});
      else fn(IC<2>{}, IC<1>{});
    } else {
      if (shape == 2) fn(IC<3>{}, IC<2>{});
      else fn(IC<3>{}, IC<1>{});
    }
  }
  double residual_up(const double* xd, double dt, double* rd) {
    if (!(dt > 0.0)) throw SimError(IMPM_ERR_CONFIG, "coupled step requires dt > 0");
    const PoroC q = poro_c();
    dispatch_up([&](auto Dc, auto Sc) {
      constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
      if (P > 0) {
        Prof::Scope ps(&prof, kcResP);
        k_up_particles<DD, SH><<<blocks_for(P), kThreads, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, orig.p, xd, q,
                                                                  Pst.p, st.p); ++g_launches;
        CKL();
      }
      Prof::Scope ps(&prof, kcResN);
      k_up_nodes<DD, SH><<<kRedBlocks, kThreads, 0, s>>>(g, pd.p, cap, xs.p, bin_start.p, sup.p, Pst.p, bext.p,
                                                         act_flag.p, freem.p, q, dt, rd, partials.p); ++g_launches;
      k_finalize_sum<1><<<1, 1024, 0, s>>>(partials.p, kRedBlocks, &st.p->norm2); ++g_launches;
      CKL();
    });
    read_status();
    prof.flush();
    if (h_st->err_domain != INT_MAX)
      throw SimError(IMPM_ERR_DOMAIN, "non-positive det(F) at particle " + std::to_string(h_st->err_domain));
    return std::sqrt(h_st->norm2);
  }

  void jacobian_up(const double* xd, double dt) {
    const PoroC q = poro_c();
    dispatch_up([&](auto Dc, auto Sc) {
      constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
      if (P > 0) {
        Prof::Scope ps(&prof, kcTangent);
        k_up_tangent<DD, SH><<<blocks_for(P, 128), 128, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, xd, q, Atan.p);
        ++g_launches;
        CKL();
      }
      if (n_act > 0) {
        Prof::Scope ps(&prof, kcAssemble);
        k_zero_rows<<<blocks_for(static_cast<int64_t>(n_act) * 32), kThreads, 0, s>>>(n_act, DD + 1, row_nzb.p, vals.p,
                                                                                    row_len); ++g_launches;
        constexpr int W = 4;
        const int nc = ipow_c(3, DD);
        for (int col = 0; col < nc; ++col) {
          int cc[3] = {0, 0, 0}, nb[3] = {1, 1, 1}, rr = col;
          for (int a = DD - 1; a >= 0; --a) {
            cc[a] = rr % 3;
            rr /= 3;
            nb[a] = std::max(0, (g.nodes[a] - cc[a] + 2) / 3);
          }
          const int nbins = nb[0] * nb[1] * nb[2];
          if (nbins == 0) continue;
          k_up_assemble_bins<DD, SH, (DD == 2 ? 3 : 2), W>
              <<<std::min<unsigned>(blocks_for(nbins, W), 148 * 16), W * 32, 0, s>>>(
                  g, pd.p, cap, xs.p, bin_start.p, bflag.p, Atan.p, act_idx.p, row_mask.p, row_nzb.p, vals.p, row_len,
                  dt * q.mob, cc[0], cc[1], cc[2], nb[0], nb[1], nb[2]); ++g_launches;
        }
        k_diag_inverse<DD, DD + 1><<<blocks_for(n_act), kThreads, 0, s>>>(n_act, act_list.p, freem.p, row_mask.p,
                                                                          row_nzb.p, vals.p, row_len, dinv.p); ++g_launches;
        CKL();
      }
    });
    matrix_valid = true;
  }

  // CoupledSim::step (src/porous.cpp:91-168): no line search, convergence on
  // |r| / (largest r0 seen), then commit F / V / sigma / p_nodes / settlement
  void coupled_step(double dt, impm_step_record* rec) {
    if (!step_built) begin_step();
    up_dt = dt;
    ++step_counter;
    std::vector<double> rels;
    const auto t0 = std::chrono::steady_clock::now();
    double diff_s = 0.0, solve_s = 0.0;
    int kry = 0, iters = 0;
    // x = (0 for u, committed nodal pressure for p), masked to free DOFs
    mask_copy(prev.p, u.p);
    double rn = residual_up(u.p, dt, r.p);
    const double r0 = rn;
    up_rscale = std::max(up_rscale, r0);
    const double denom = up_rscale;
    bool converged = r0 < opt.abs_floor;
    for (int it = 1; it <= opt.max_iterations && !converged; ++it) {
      auto tj = std::chrono::steady_clock::now();
      jacobian_up(u.p, dt);
      sync();
      diff_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tj).count();
      auto ts = std::chrono::steady_clock::now();
      axpbypcz(-1.0, r.p, 0.0, tmp2.p);
      // forcing term against the reference's convergence scale (porous.cpp:
      // 105-110, 135): |J d + r| <= 1% of tol * r_scale adds at most 1% of the
      // Newton tolerance to the next residual. Warm-started steps begin with
      // |r| << r_scale, where a relative 1e-12 of |r| is below the attainable
      // accuracy of the saddle point (cond ~1e15); floor = krylov_rtol.
      cur_rtol = std::min(1e-6, std::max(opt.krylov_rtol, 0.01 * opt.tol * denom / std::max(rn, 1e-300)));
      kry += solve_dev(tmp2.p, delta.p);
      cur_rtol = opt.krylov_rtol;
      solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
      axpbypcz(1.0, delta.p, 1.0, u.p);
      rn = residual_up(u.p, dt, r.p);
      rels.push_back(rn / denom);
      iters = it;
      if (rn / denom <= opt.tol || rn < opt.abs_floor) converged = true;
    }
    if (rec) {
      rec->step = step_counter;
      rec->iterations = iters;
      rec->r0_norm = r0;
      rec->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      rec->diff_seconds = diff_s;
      rec->solve_seconds = solve_s;
      rec->krylov_iterations = kry;
      rec->backward_passes = iters * (opt.strategy == IMPM_STRATEGY_DENSE ? ndg() : F * (D == 2 ? 25 : 125));
      rec->nnz_assembled = iters * ref_nnz();
      finish_record(rec, rels);
    }
    if (!converged)
      throw SimError(IMPM_ERR_NONCONVERGENCE, "coupled Newton did not converge at step " + std::to_string(step_counter),
                     rels);
    // commit (src/porous.cpp:139-163)
    const PoroC q = poro_c();
    if (P > 0) {
      Prof::Scope ps(&prof, kcCommit);
      dispatch_up([&](auto Dc, auto Sc) {
        constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
        k_up_commit<DD, SH><<<blocks_for(P), kThreads, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, u.p, q, uty.p);
      });
      ++g_launches;
      CKL();
    }
    // p_nodes <- pressure DOFs of x (displacement components are not kept)
    CK(cudaMemsetAsync(prev.p, 0, sizeof(double) * NF(), s));
    k_copy_field<<<blocks_for(g.N), kThreads, 0, s>>>(g.N, F, D, freem.p, u.p, prev.p); ++g_launches;
    CKL();
    up_time += dt;
    sync();
  }
  // ------------------------------------------------------- commit (K9)
  void commit_step() {
    if (!step_built) throw SimError(IMPM_ERR_CONFIG, "commit_step before begin_step");
    clear_errors_only();
    const int big = INT_MAX;
    CK(cudaMemcpyAsync(&st.p->err_lp, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    halo(u.p);
    const MatParams mp = matp();
    dispatch([&](auto Dc, auto Sc) {
      constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
      if (P > 0) {
        Prof::Scope ps(&prof, kcCommit);
        if (mp.kind == kNeoHookean)
          k_commit<DD, SH, true><<<blocks_for(P), kThreads, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, orig.p, u.p,
                                                                    mp, opt.total_lagrangian, st.p);
        else
          k_commit<DD, SH, false><<<blocks_for(P), kThreads, 0, s>>>(g, pd.p, cap, P, xs.p, key.p, sup.p, orig.p, u.p,
                                                                     mp, opt.total_lagrangian, st.p);
        ++g_launches;
        CKL();
      }
    });
    gmin_int(&st.p->err_domain, 5);  // err_domain .. err_lp
    read_status();
    prof.flush();
    if (h_st->err_domain != INT_MAX)
      throw SimError(IMPM_ERR_DOMAIN, "inverted element at particle " + std::to_string(h_st->err_domain) +
                                          ": det(I + grad du) <= 0");
    if (h_st->err_lp != INT_MAX)
      throw SimError(IMPM_ERR_DOMAIN, "particle domain half-width of particle " + std::to_string(h_st->err_lp) +
                                          " reached half the grid spacing " + std::to_string(g.h) +
                                          "; use finer particles or a capped domain update");
    if (!opt.total_lagrangian) step_built = false;  // grid reset
  }

  // ------------------------------------------------------- parity taps
  void upload_dof_vec(const double* h, double* gvec) {
    CK(cudaMemsetAsync(gvec, 0, sizeof(double) * NF(), s));
    if (n_dofs == 0) return;
    CK(cudaMemcpyAsync(kt.p, h, sizeof(double) * n_dofs, cudaMemcpyHostToDevice, s));
    k_dof_to_grid<<<blocks_for(n_dofs), kThreads, 0, s>>>(n_dofs, kt.p, node_of.p, field_of.p, F, gvec); ++g_launches;
    CKL();
  }
  void download_dof_vec(const double* gvec, double* h) {
    if (n_dofs == 0) return;
    k_grid_to_dof<<<blocks_for(n_dofs), kThreads, 0, s>>>(n_dofs, gvec, node_of.p, field_of.p, F, kt.p); ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(h, kt.p, sizeof(double) * n_dofs, cudaMemcpyDeviceToHost, s));
    sync();
  }

  void export_csr(int64_t* nnz, int64_t* row_ptr_h, int32_t* cols_h, double* vals_h) {
    const int64_t z = ref_nnz();
    *nnz = z;
    if (!row_ptr_h) return;
    std::vector<int64_t> rl(n_dofs);
    if (n_dofs) CK(cudaMemcpyAsync(rl.data(), rowlen.p, sizeof(int64_t) * n_dofs, cudaMemcpyDeviceToHost, s));
    sync();
    row_ptr_h[0] = 0;
    for (int i = 0; i < n_dofs; ++i) row_ptr_h[i + 1] = row_ptr_h[i] + rl[i];
    if (n_dofs == 0) return;
    CK(cudaMemcpyAsync(rowptr.p, row_ptr_h, sizeof(int64_t) * (n_dofs + 1), cudaMemcpyHostToDevice, s));
    DBuf<int> dcols;
    DBuf<double> dvals;
    dcols.ensure(z);
    dvals.ensure(z);
    dispatch_df([&](auto Dc, auto Fc) {
      constexpr int DD = decltype(Dc)::value, FE = decltype(Fc)::value;
      k_csr_fill<DD, FE><<<blocks_for(n_dofs), kThreads, 0, s>>>(g, n_dofs, node_of.p, field_of.p, dof_of.p, act_idx.p,
                                                                 vals.p, row_len, row_slots.p, row_nzb.p, rowptr.p,
                                                                 dcols.p,
                                                                 vals_h ? dvals.p : nullptr); ++g_launches;
      CKL();
    });
    if (cols_h) CK(cudaMemcpyAsync(cols_h, dcols.p, sizeof(int32_t) * z, cudaMemcpyDeviceToHost, s));
    if (vals_h) CK(cudaMemcpyAsync(vals_h, dvals.p, sizeof(double) * z, cudaMemcpyDeviceToHost, s));
    sync();
  }
};

impm_status fail(Sim* sim, const SimError& e) {
  if (sim) {
    sim->err_msg = e.what();
    sim->err_hist = e.history;
  }
  return e.code;
}

thread_local std::string g_create_error;

}  // namespace

namespace {
thread_local std::string g_csr_error;

// Runs one CSR call on `device` on a private stream; errors -> g_csr_error.
template <class F>
impm_status csr_call(int32_t device, F&& f) {
  cudaStream_t s = nullptr;
  try {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    f(s);
    cudaStreamDestroy(s);
    g_csr_error.clear();
    return IMPM_OK;
  } catch (const SimError& e) {
    if (s) cudaStreamDestroy(s);
    g_csr_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (s) cudaStreamDestroy(s);
    g_csr_error = e.what();
    return IMPM_ERR_CUDA;
  }
}
}  // namespace

// opaque communicator handle of the C ABI (include/impm_gpu.h)
struct impm_comm {
  std::shared_ptr<Comm> c;
};

// ================================================================ C ABI ===
#define API_BEGIN(sim)        \
  if (!(sim)) return IMPM_ERR_CONFIG; \
  try {                       \
    CK(cudaSetDevice((sim)->device));
#define API_END(sim)                                            \
  return IMPM_OK;                                               \
  }                                                             \
  catch (const SimError& e) {                                   \
    return fail(sim, e);                                        \
  }                                                             \
  catch (const std::exception& e) {                             \
    return fail(sim, SimError(IMPM_ERR_CUDA, e.what()));        \
  }

extern "C" {

const char* impm_version(void) { return "impm-b200 0.1 (sm_100a, fp64)"; }
int64_t impm_launch_count(void) { return g_launches.load(); }
int32_t impm_particle_doubles(int32_t dim) { return 6 * dim + 22 + dim * dim; }

impm_status impm_sim_create(const impm_grid* grid, const impm_material* mat, const impm_options* opt, int32_t device,
                            impm_sim** out) {
  if (!grid || !mat || !opt || !out) return IMPM_ERR_CONFIG;
  try {
    *out = reinterpret_cast<impm_sim*>(new Sim(grid, mat, opt, device));
    return IMPM_OK;
  } catch (const SimError& e) {
    g_create_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return IMPM_ERR_CUDA;
  }
}

const char* impm_create_error(void) { return g_create_error.c_str(); }

impm_status impm_coupled_create(const impm_grid* grid, const impm_poro* poro, const impm_options* opt, int32_t device,
                                impm_sim** out) {
  if (!grid || !poro || !opt || !out) return IMPM_ERR_CONFIG;
  try {
    impm_material dummy{IMPM_NEO_HOOKEAN, 0, 1.0, 0.0, 0.0, 30.0, 0.0};
    *out = reinterpret_cast<impm_sim*>(new Sim(grid, &dummy, opt, device, poro));
    return IMPM_OK;
  } catch (const SimError& e) {
    g_create_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return IMPM_ERR_CUDA;
  }
}

impm_status impm_sim_destroy(impm_sim* h) {
  delete reinterpret_cast<Sim*>(h);
  return IMPM_OK;
}

#define SIM Sim* sim = reinterpret_cast<Sim*>(h)

impm_status impm_sim_set_stream(impm_sim* h, void* stream) {
  SIM;
  API_BEGIN(sim)
  sim->s = stream ? static_cast<cudaStream_t>(stream) : sim->own_stream;
  sim->prof.s = sim->s;
  API_END(sim)
}

impm_status impm_sim_set_particles(impm_sim* h, const double* aos, int64_t n, int64_t stride) {
  SIM;
  API_BEGIN(sim)
  sim->set_particles(aos, n, stride);
  API_END(sim)
}
impm_status impm_sim_get_particles(impm_sim* h, double* aos, int64_t n, int64_t stride) {
  SIM;
  API_BEGIN(sim)
  sim->get_particles(aos, n, stride);
  API_END(sim)
}
impm_status impm_sim_set_particle_field(impm_sim* h, int32_t field, const double* vals) {
  SIM;
  API_BEGIN(sim)
  sim->set_particle_field(field, vals);
  API_END(sim)
}
impm_status impm_sim_n_particles(impm_sim* h, int64_t* n) {
  SIM;
  API_BEGIN(sim)
  *n = sim->P;
  API_END(sim)
}
impm_status impm_sim_set_fixed(impm_sim* h, const uint8_t* fixed) {
  SIM;
  API_BEGIN(sim)
  CK(cudaMemcpyAsync(sim->fixed.p, fixed, sim->NF(), cudaMemcpyHostToDevice, sim->s));
  sim->sync();
  sim->step_built = sim->opt.total_lagrangian ? sim->step_built : false;
  API_END(sim)
}
impm_status impm_sim_set_gravity(impm_sim* h, const double* gv) {
  SIM;
  API_BEGIN(sim)
  for (int a = 0; a < 3; ++a) sim->gravity[a] = a < sim->D ? gv[a] : 0.0;
  API_END(sim)
}
impm_status impm_sim_set_options(impm_sim* h, const impm_options* o) {
  SIM;
  API_BEGIN(sim)
  sim->set_options(o);
  API_END(sim)
}
impm_status impm_sim_begin_step(impm_sim* h) {
  SIM;
  API_BEGIN(sim)
  sim->begin_step();
  API_END(sim)
}
impm_status impm_sim_n_dofs(impm_sim* h, int32_t* n) {
  SIM;
  API_BEGIN(sim)
  *n = sim->n_dofs;
  API_END(sim)
}
impm_status impm_sim_dof_map(impm_sim* h, int32_t* dof_of, int32_t* node_of, int32_t* field_of) {
  SIM;
  API_BEGIN(sim)
  if (dof_of) CK(cudaMemcpyAsync(dof_of, sim->dof_of.p, sizeof(int) * sim->NF(), cudaMemcpyDeviceToHost, sim->s));
  if (node_of && sim->n_dofs)
    CK(cudaMemcpyAsync(node_of, sim->node_of.p, sizeof(int) * sim->n_dofs, cudaMemcpyDeviceToHost, sim->s));
  if (field_of && sim->n_dofs)
    CK(cudaMemcpyAsync(field_of, sim->field_of.p, sizeof(int) * sim->n_dofs, cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  API_END(sim)
}
impm_status impm_sim_node_mass(impm_sim* h, double* m) {
  SIM;
  API_BEGIN(sim)
  CK(cudaMemcpyAsync(m, sim->mass.p, sizeof(double) * sim->g.N, cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  API_END(sim)
}
impm_status impm_sim_colour_groups(impm_sim* h, int32_t* group_of_dof, int32_t* n_groups) {
  SIM;
  API_BEGIN(sim)
  // group = field * 5^D + sum_a (idx_a mod 5) 5^(D-1-a)   (jacobian.hpp:101-110)
  const int S = ipow_c(5, sim->D);
  *n_groups = sim->F * S;
  if (group_of_dof && sim->n_dofs) {
    std::vector<int> node_of(sim->n_dofs), field_of(sim->n_dofs);
    CK(cudaMemcpyAsync(node_of.data(), sim->node_of.p, sizeof(int) * sim->n_dofs, cudaMemcpyDeviceToHost, sim->s));
    CK(cudaMemcpyAsync(field_of.data(), sim->field_of.p, sizeof(int) * sim->n_dofs, cudaMemcpyDeviceToHost, sim->s));
    sim->sync();
    for (int d = 0; d < sim->n_dofs; ++d) {
      int off = 0;
      for (int a = 0; a < sim->D; ++a) off = off * 5 + ((node_of[d] / sim->g.stride[a]) % sim->g.nodes[a]) % 5;
      group_of_dof[d] = field_of[d] * S + off;
    }
  }
  API_END(sim)
}
int64_t impm_debug_oob_count(void) {
#ifdef IMPM_CHECKED
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, impm_gpu::g_oob_count, sizeof(v)) != cudaSuccess) return -2;
  return static_cast<int64_t>(v);
#else
  return -1;
#endif
}
impm_status impm_sim_support_stats(impm_sim* h, int64_t* out) {
  SIM;
  API_BEGIN(sim)
  // [P, sum s_p, sum s_p^2, sum_bins n_p * nk, sum_bins n_p * nk^2, bins, histogram of s_p (1..27)]
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "support_stats before begin_step");
  const int P = sim->P, N = sim->g.N;
  std::vector<int> sup(std::max(P, 1)), bs(N + 1);
  std::vector<uint8_t> bf(std::max(N, 1));
  CK(cudaMemcpyAsync(sup.data(), sim->sup.p, sizeof(int) * P, cudaMemcpyDeviceToHost, sim->s));
  CK(cudaMemcpyAsync(bs.data(), sim->bin_start.p, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost, sim->s));
  CK(cudaMemcpyAsync(bf.data(), sim->bflag.p, N, cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  for (int i = 0; i < 34; ++i) out[i] = 0;
  out[0] = P;
  for (int p = 0; p < P; ++p) {
    int sp = 1;
    for (int a = 0; a < sim->D; ++a) sp *= (sup[p] >> (2 * a)) & 3;
    out[1] += sp;
    out[2] += static_cast<int64_t>(sp) * sp;
    if (sp <= 27) out[6 + sp] += 1;
  }
  for (int b = 0; b < N; ++b) {
    const int np = bs[b + 1] - bs[b];
    if (np == 0) continue;
    int nk = 1;
    for (int a = 0; a < sim->D; ++a) nk *= 2 + ((bf[b] >> a) & 1);
    out[3] += static_cast<int64_t>(np) * nk;
    out[4] += static_cast<int64_t>(np) * nk * nk;
    out[5] += 1;
  }
  API_END(sim)
}
impm_status impm_sim_p2g_map(impm_sim* h, const double* per_particle, double* out) {
  SIM;
  API_BEGIN(sim)
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "p2g_map before begin_step");
  DBuf<double> f, o;
  f.ensure(std::max(sim->P, 1));
  o.ensure(sim->g.N);
  DBuf<double> fo;
  fo.ensure(std::max(sim->P, 1));
  CK(cudaMemcpyAsync(fo.p, per_particle, sizeof(double) * sim->P, cudaMemcpyHostToDevice, sim->s));
  k_set_field<<<blocks_for(sim->P), kThreads, 0, sim->s>>>(f.p, fo.p, sim->orig.p, sim->P); ++g_launches;
  sim->dispatch([&](auto Dc, auto Sc) {
    constexpr int DD = decltype(Dc)::value, SH = decltype(Sc)::value;
    k_p2g_map<DD, SH><<<blocks_for(sim->g.N), kThreads, 0, sim->s>>>(sim->g, sim->pd.p, sim->cap, sim->xs.p,
                                                                      sim->bin_start.p, sim->sup.p, sim->mass.p, f.p,
                                                                      o.p); ++g_launches;
  });
  CKL();
  CK(cudaMemcpyAsync(out, o.p, sizeof(double) * sim->g.N, cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  API_END(sim)
}
impm_status impm_sim_residual(impm_sim* h, const double* uh, double load_scale, double* rh) {
  SIM;
  API_BEGIN(sim)
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "residual before begin_step");
  sim->upload_dof_vec(uh, sim->tmp1.p);
  sim->residual_dev(sim->tmp1.p, load_scale, sim->rtry.p);
  sim->download_dof_vec(sim->rtry.p, rh);
  API_END(sim)
}
impm_status impm_sim_jacobian_csr(impm_sim* h, const double* uh, double load_scale, int64_t* nnz, int64_t* row_ptr,
                                  int32_t* cols, double* vals) {
  SIM;
  API_BEGIN(sim)
  // J does not depend on the load scale (external loads are constant in u);
  // in coupled mode the argument is the time step dt (K_pp = V0 dt mob g.g)
  if (sim->coupled) sim->up_dt = load_scale;
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "jacobian before begin_step");
  if (row_ptr && uh) {
    sim->upload_dof_vec(uh, sim->tmp1.p);
    sim->jacobian_dev(sim->tmp1.p);
    sim->sync();
    sim->prof.flush();
  }
  sim->export_csr(nnz, row_ptr, cols, vals);
  API_END(sim)
}
impm_status impm_sim_linear_solve(impm_sim* h, const double* uh, double load_scale, const double* rhs, double* delta,
                                  int32_t* kit) {
  SIM;
  API_BEGIN(sim)
  if (sim->coupled) sim->up_dt = load_scale;
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "linear_solve before begin_step");
  sim->upload_dof_vec(uh, sim->tmp1.p);
  sim->jacobian_dev(sim->tmp1.p);
  sim->upload_dof_vec(rhs, sim->tmp2.p);
  const int it = sim->solve_dev(sim->tmp2.p, sim->delta.p);
  if (kit) *kit = it;
  sim->download_dof_vec(sim->delta.p, delta);
  sim->prof.flush();
  API_END(sim)
}
impm_status impm_sim_newton_solve(impm_sim* h, double load_scale, impm_step_record* rec) {
  SIM;
  API_BEGIN(sim)
  sim->newton_solve(load_scale, rec);
  API_END(sim)
}
impm_status impm_sim_commit_step(impm_sim* h) {
  SIM;
  API_BEGIN(sim)
  sim->commit_step();
  API_END(sim)
}
impm_status impm_sim_step(impm_sim* h, double load_scale, impm_step_record* rec) {
  SIM;
  API_BEGIN(sim)
  sim->begin_step();
  sim->newton_solve(load_scale, rec);
  sim->commit_step();
  if (sim->slab) sim->migrate();  // particles follow their slab for the next step
  API_END(sim)
}
impm_status impm_coupled_initialize(impm_sim* h) {
  SIM;
  API_BEGIN(sim)
  if (!sim->coupled) throw SimError(IMPM_ERR_CONFIG, "not a coupled simulation");
  sim->begin_step();
  API_END(sim)
}
impm_status impm_coupled_step(impm_sim* h, double dt, impm_step_record* rec) {
  SIM;
  API_BEGIN(sim)
  if (!sim->coupled) throw SimError(IMPM_ERR_CONFIG, "not a coupled simulation");
  sim->coupled_step(dt, rec);
  API_END(sim)
}
impm_status impm_coupled_nodal_pressure(impm_sim* h, double* p) {
  SIM;
  API_BEGIN(sim)
  if (!sim->coupled) throw SimError(IMPM_ERR_CONFIG, "not a coupled simulation");
  std::vector<double> gv(sim->NF());
  CK(cudaMemcpyAsync(gv.data(), sim->prev.p, sizeof(double) * gv.size(), cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  for (int n = 0; n < sim->g.N; ++n) p[n] = gv[static_cast<size_t>(n) * sim->F + sim->D];
  API_END(sim)
}
impm_status impm_coupled_settlement(impm_sim* h, double* u_total_y, double* time) {
  SIM;
  API_BEGIN(sim)
  if (!sim->coupled) throw SimError(IMPM_ERR_CONFIG, "not a coupled simulation");
  if (time) *time = sim->up_time;
  if (u_total_y && sim->P > 0) {
    DBuf<double> o;
    o.ensure(sim->P);
    k_gather_orig<<<blocks_for(sim->P), kThreads, 0, sim->s>>>(sim->uty.p, sim->orig.p, sim->P, o.p); ++g_launches;
    CKL();
    CK(cudaMemcpyAsync(u_total_y, o.p, sizeof(double) * sim->P, cudaMemcpyDeviceToHost, sim->s));
    sim->sync();
  }
  API_END(sim)
}

impm_status impm_sim_nodal_solution(impm_sim* h, double* uh) {
  SIM;
  API_BEGIN(sim)
  sim->download_dof_vec(sim->u.p, uh);
  API_END(sim)
}
impm_status impm_sim_set_nodal_solution(impm_sim* h, const double* uh) {
  SIM;
  API_BEGIN(sim)
  sim->upload_dof_vec(uh, sim->u.p);
  sim->sync();
  API_END(sim)
}
impm_status impm_sim_last_error(impm_sim* h, char* msg, size_t cap, double* history, int32_t* hist_len) {
  SIM;
  if (!sim) {
    if (msg && cap) std::snprintf(msg, cap, "%s", g_create_error.c_str());
    return IMPM_OK;
  }
  if (msg && cap) std::snprintf(msg, cap, "%s", sim->err_msg.c_str());
  if (hist_len) {
    const int n = static_cast<int>(sim->err_hist.size());
    if (history)
      for (int i = 0; i < std::min(n, *hist_len); ++i) history[i] = sim->err_hist[i];
    *hist_len = n;
  }
  return IMPM_OK;
}
impm_status impm_sim_kernel_times(impm_sim* h, const char** names, double* ms, int64_t* launches, int32_t* n,
                                  int32_t reset) {
  SIM;
  API_BEGIN(sim)
  sim->sync();
  sim->prof.flush();
  *n = kcCount;
  for (int i = 0; i < kcCount; ++i) {
    if (names) names[i] = kClassNames[i];
    if (ms) ms[i] = sim->prof.ms[i];
    if (launches) launches[i] = sim->prof.launches[i];
  }
  if (reset) {
    for (int i = 0; i < kcCount; ++i) {
      sim->prof.ms[i] = 0;
      sim->prof.launches[i] = 0;
    }
  }
  API_END(sim)
}
impm_status impm_sim_matrix_info(impm_sim* h, int64_t* n_rows, int64_t* row_values, int64_t* ref_nnz) {
  SIM;
  API_BEGIN(sim)
  if (n_rows) *n_rows = sim->n_act;
  if (row_values) {
    sim->sync();
    *row_values = static_cast<int64_t>(sim->h_nzb_total) * sim->F * sim->F;  // stored block values (all rows)
  }
  if (ref_nnz) *ref_nnz = sim->step_built ? sim->ref_nnz() : 0;
  API_END(sim)
}

// ------------------------------------------------- slab decomposition (§8e)
impm_status impm_comm_nccl_id(uint8_t* id, int32_t cap) {
  if (!id || cap < static_cast<int32_t>(sizeof(ncclUniqueId))) return IMPM_ERR_CONFIG;
  ncclUniqueId u;
  const ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return IMPM_ERR_NCCL;
  }
  std::memcpy(id, &u, sizeof(u));
  return IMPM_OK;
}
impm_status impm_comm_nccl_create(const uint8_t* id, int32_t rank, int32_t nranks, int32_t device, impm_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return IMPM_ERR_CONFIG;
  try {
    CK(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    *out = new impm_comm{std::make_shared<NcclComm>(u, rank, nranks)};
    return IMPM_OK;
  } catch (const CommError& e) {
    g_create_error = e.what();
    return IMPM_ERR_NCCL;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return IMPM_ERR_CUDA;
  }
}
impm_status impm_comm_local_group(int32_t nranks, int32_t device, impm_comm** out) {
  if (!out || nranks < 1) return IMPM_ERR_CONFIG;
  try {
    CK(cudaSetDevice(device));
    auto grp = std::make_shared<LocalGroup>(nranks);
    for (int r = 0; r < nranks; ++r) out[r] = new impm_comm{std::make_shared<LocalComm>(grp, r)};
    return IMPM_OK;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return IMPM_ERR_CUDA;
  }
}
impm_status impm_comm_destroy(impm_comm* c) {
  delete c;
  return IMPM_OK;
}
impm_status impm_comm_info(impm_comm* c, int32_t* rank, int32_t* nranks, const char** kind) {
  if (!c) return IMPM_ERR_CONFIG;
  if (rank) *rank = c->c->rank;
  if (nranks) *nranks = c->c->nranks;
  if (kind) *kind = c->c->kind();
  return IMPM_OK;
}
impm_status impm_sim_set_slab(impm_sim* h, impm_comm* c, int32_t global_n0, const int32_t* cuts) {
  SIM;
  API_BEGIN(sim)
  if (!c || !cuts) throw SimError(IMPM_ERR_CONFIG, "set_slab needs a communicator and the ownership cuts");
  sim->set_slab(c->c, global_n0, cuts);
  API_END(sim)
}
impm_status impm_sim_set_particles_ids(impm_sim* h, const double* aos, const int64_t* ids, int64_t n, int64_t stride) {
  SIM;
  API_BEGIN(sim)
  sim->set_particles_ids(aos, ids, n, stride);
  API_END(sim)
}
impm_status impm_sim_get_particles_ids(impm_sim* h, double* aos, int64_t* ids, int64_t n, int64_t stride) {
  SIM;
  API_BEGIN(sim)
  sim->get_particles_ids(aos, ids, n, stride);
  API_END(sim)
}
impm_status impm_sim_migrate(impm_sim* h) {
  SIM;
  API_BEGIN(sim)
  sim->migrate();
  API_END(sim)
}
impm_status impm_sim_slab_info(impm_sim* h, int64_t* n_dofs_global, int64_t* dof_offset, int32_t* base0) {
  SIM;
  API_BEGIN(sim)
  if (n_dofs_global) *n_dofs_global = sim->n_dofs_glob;
  if (dof_offset) *dof_offset = sim->dof_offset;
  if (base0) *base0 = sim->g.base0;
  API_END(sim)
}
impm_status impm_sim_apply_jacobian(impm_sim* h, const double* uh, double load_scale, const double* x, double* y) {
  SIM;
  API_BEGIN(sim)
  (void)load_scale;  // J does not depend on the load scale (external loads are constant in u)
  if (!sim->step_built) throw SimError(IMPM_ERR_CONFIG, "apply_jacobian before begin_step");
  if (sim->coupled) throw SimError(IMPM_ERR_UNSUPPORTED, "apply_jacobian: single-field simulations only");
  sim->upload_dof_vec(uh, sim->tmp1.p);
  sim->jacobian_dev(sim->tmp1.p);
  const int64_t nf = sim->NF();
  CK(cudaMemcpyAsync(sim->kx.p, x, sizeof(double) * nf, cudaMemcpyHostToDevice, sim->s));
  CK(cudaMemsetAsync(sim->kq.p, 0, sizeof(double) * nf, sim->s));
  sim->spmv(sim->kx.p, sim->kq.p, nullptr, nullptr);
  CK(cudaMemcpyAsync(y, sim->kq.p, sizeof(double) * nf, cudaMemcpyDeviceToHost, sim->s));
  sim->sync();
  sim->prof.flush();
  API_END(sim)
}

// ---- link-level seam: impm::sparse_lu_solve / CsrMatrix (impm_csr.cuh) ----
impm_status impm_sparse_lu_solve(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                                 const double* b, int64_t b_len, double* x, int32_t device, int32_t* iterations) {
  if (n == 0) return IMPM_OK;  // linear_solver.cpp:12
  if (b_len != n) {            // :13-14
    g_csr_error = "right-hand side size does not match the matrix dimension";
    return IMPM_ERR_LINEAR_SOLVER;
  }
  if (!row_ptr || !cols || !vals || !b || !x) {
    g_csr_error = "null pointer argument";
    return IMPM_ERR_CONFIG;
  }
  return csr_call(device, [&](cudaStream_t s) {
    csr::LuSolver lu;
    lu.A.upload(n, row_ptr, cols, vals, s);
    lu.solve(b, x);
    if (iterations) *iterations = lu.A.n <= csr::kDenseMax ? 0 : lu.krylov_iterations;
  });
}
impm_status impm_csr_multiply(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                              const double* x, double* y, int32_t device) {
  if (n == 0) return IMPM_OK;
  return csr_call(device, [&](cudaStream_t s) {
    csr::DevCsr A;
    A.upload(n, row_ptr, cols, vals, s);
    DBuf<double> dx, dy;
    dx.ensure(n);
    dy.ensure(n);
    CK(cudaMemcpyAsync(dx.get(), x, n * sizeof(double), cudaMemcpyHostToDevice, s));
    A.spmv<0>(dx.get(), dy.get());
    CK(cudaMemcpyAsync(y, dy.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}
impm_status impm_csr_transposed(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                                int64_t* t_row_ptr, int32_t* t_cols, double* t_vals, int32_t device) {
  if (n == 0) {
    if (t_row_ptr) t_row_ptr[0] = 0;
    return IMPM_OK;
  }
  return csr_call(device, [&](cudaStream_t s) {
    csr::DevCsr A;
    A.upload(n, row_ptr, cols, vals, s);
    csr::transposed(A, t_row_ptr, t_cols, t_vals);
  });
}
const char* impm_csr_last_error(void) { return g_csr_error.c_str(); }

}  // extern "C"
