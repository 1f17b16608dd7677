// strips.cu -- row-strip partitioned multigrid-ORAS solve.
//
// One image is cut into P horizontal strips.  Each strip owns rows [o0, o1)
// of every partitioned level (the finest La levels) and computes on a view
// [e0, e1) = owned rows widened by `halo` rows on each side.  A strip keeps a
// full-size hierarchy (180 GB of HBM makes that the simple layout); only its
// view rows are ever computed, so per-strip work is O(H/P).  The coarse
// levels >= La are replicated: every strip gathers the restricted residual
// of level La and runs the identical coarse V-cycle (agglomeration).
//
// Per smoothing sweep of a partitioned level:
//   exchange u halo (neighbours' owned rows) -> residual on the view ->
//   per-(16-row band, 128-column group) partial sum r^2 -> owned bands summed
//   -> band sums gathered from every strip -> per-channel norm summed over
//   bands in index order -> ORAS local CG on the blocks inside the view ->
//   blend on the view.
// The view edges act as image boundaries, so results are wrong within 32
// rows of an artificial edge -- inside the halo, never on owned rows (halo
// = 48 >= block 32 + stencil 1); exchanges refresh the halo before each use.
// The band partials are independent of the partition, so the solve is
// bit-identical for every P (tests/test_strips_gpu.py).
//
// Transport: strips held by this process exchange through device copies
// ("loopback": P logical strips on one GPU, the single-GPU test harness);
// strips on other ranks through NCCL point-to-point sends / receives
// (halo rows), all-reduce of zero-padded band sums and broadcasts (row
// gathers), each batch inside one ncclGroupStart/End.  NCCL is dlopen'd:
// the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <vector>

#include "kernels.cuh"
#include "solver.cuh"

namespace sp {

void cover_tables(const std::vector<int>& starts, int size, int dim, std::vector<int>& k0,
                  std::vector<int>& n);

// ---- NCCL through dlopen --------------------------------------------------------
namespace {
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId;
  decltype(&ncclCommInitRank) CommInitRank;
  decltype(&ncclCommDestroy) CommDestroy;
  decltype(&ncclSend) Send;
  decltype(&ncclRecv) Recv;
  decltype(&ncclAllReduce) AllReduce;
  decltype(&ncclBroadcast) Broadcast;
  decltype(&ncclGroupStart) GroupStart;
  decltype(&ncclGroupEnd) GroupEnd;
  decltype(&ncclGetErrorString) GetErrorString;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define SP_SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
  SP_SYM(GetUniqueId);
  SP_SYM(CommInitRank);
  SP_SYM(CommDestroy);
  SP_SYM(Send);
  SP_SYM(Recv);
  SP_SYM(AllReduce);
  SP_SYM(Broadcast);
  SP_SYM(GroupStart);
  SP_SYM(GroupEnd);
  SP_SYM(GetErrorString);
#undef SP_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
           api.AllReduce && api.Broadcast && api.GroupStart && api.GroupEnd &&
           api.GetErrorString;
  return api.ok ? &api : nullptr;
}
}  // namespace

#define SP_NCCL(expr)                                                           \
  do {                                                                          \
    ncclResult_t _r = (expr);                                                   \
    if (_r != ncclSuccess) {                                                    \
      ::sp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                \
                      nccl()->GetErrorString(_r));                              \
      return -1;                                                                \
    }                                                                           \
  } while (0)

int nccl_unique_id(uint8_t* out) {
  NcclApi* n = nccl();
  if (!n) { set_error("libnccl.so.2 not loadable"); return -1; }
  ncclUniqueId id;
  SP_NCCL(n->GetUniqueId(&id));
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int nccl_comm_create(void** comm, const uint8_t* id_bytes, int nranks, int rank) {
  NcclApi* n = nccl();
  if (!n) { set_error("libnccl.so.2 not loadable"); return -1; }
  ncclUniqueId id;
  memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c;
  SP_NCCL(n->CommInitRank(&c, nranks, id, rank));
  *comm = (void*)c;
  return 0;
}

int nccl_comm_destroy(void* comm) {
  NcclApi* n = nccl();
  if (n && comm) n->CommDestroy((ncclComm_t)comm);
  return 0;
}

// ---- the strip group ------------------------------------------------------------
struct StripView {
  int e0, e1, o0, o1;  // view rows and owned rows (level coordinates)
  int kya, nby;        // level block rows fully inside the view
  int *ys, *row_k0, *row_n;  // device tables local to the view
};

struct StripGroup {
  int P = 1, nloc = 1, first = 0, La = 0, halo = 48, C = 1, H = 0, W = 0;
  std::vector<Hier*> h;                       // [nloc] full-size hierarchies
  std::vector<std::vector<StripView>> v;      // [nloc][La]
  std::vector<std::vector<int>> o0, o1;       // [La][P] owned rows of every strip
  std::vector<int> nbt, ncg;                  // per partitioned level: bands, col groups
  std::vector<std::vector<double*>> bandcol;  // [nloc][La] [C][nbt][ncg]
  std::vector<std::vector<double*>> bands;    // [nloc][La] [C][nbt]
  ncclComm_t comm = nullptr;                  // strips on other ranks (P > nloc)
  // host-staged transport (sp_strip_set_host_transport): the same exchanges
  // through caller callbacks on pinned host buffers, stream-synchronous and
  // never graph-captured -- the harness that runs the multi-rank protocol
  // where NCCL cannot (several ranks on one GPU)
  HostTransport host{};
  bool host_mode = false;
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // the V-cycle (kernels, halo copies / NCCL calls) recorded once as a CUDA
  // graph on a private stream and replayed on the caller's stream
  cudaGraphExec_t graph = nullptr;
  cudaStream_t cap = nullptr;
  long long graph_nodes = 0;
  ~StripGroup() {
    if (graph) cudaGraphExecDestroy(graph);
    if (cap) cudaStreamDestroy(cap);
    for (auto& vs : v)
      for (auto& w : vs)
        for (int* p : {w.ys, w.row_k0, w.row_n})
          if (p) cudaFree(p);
    for (auto& vv : bandcol)
      for (double* p : vv) if (p) cudaFree(p);
    for (auto& vv : bands)
      for (double* p : vv) if (p) cudaFree(p);
    for (Hier* x : h) delete x;
    if (stage) cudaFreeHost(stage);
  }
  bool remote_ok() const { return comm != nullptr || host_mode; }
  bool local(int p) const { return p >= first && p < first + nloc; }
  int rank_of(int p) const { return p; }  // NCCL: one strip per rank, rank = strip
};

namespace {

__global__ void k_band_sum(const double* __restrict__ bandcol, double* __restrict__ bands,
                           int C, int nbt, int ncg, int b_lo, int b_hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C * nbt) return;
  const int b = i % nbt;
  double s = 0.0;
  if (b >= b_lo && b < b_hi)
    for (int g = 0; g < ncg; ++g) s += bandcol[(size_t)i * ncg + g];
  bands[i] = s;  // bands owned elsewhere contribute an exact +0
}

__global__ void k_band_total(const double* __restrict__ bands, double* __restrict__ norms,
                             int C, int nbt) {
  const int c = threadIdx.x;
  if (c >= C) return;
  double s = 0.0;
  for (int b = 0; b < nbt; ++b) s += bands[(size_t)c * nbt + b];
  norms[c] = s;
}

inline float* rowp(void* base, const Level& L, int c, int row) {
  return (float*)base + (size_t)c * L.H * L.W + (size_t)row * L.W;
}
inline uint8_t* mrow(const Level& L, int row) { return L.mask + (size_t)row * L.W; }

// ---- transport ----------------------------------------------------------------
// copy rows [r0, r1) of every channel plane of `lv`'s buffer from strip q to p
int copy_rows(StripGroup& g, int lv, int which, int p, int q, int r0, int r1, cudaStream_t s) {
  if (r1 <= r0) return 0;
  Level& Lp = g.h[p - g.first]->lv[lv];
  Level& Lq = g.h[q - g.first]->lv[lv];
  void* dst = which == 0 ? Lp.u : (which == 1 ? Lp.b : Lp.r);
  void* src = which == 0 ? Lq.u : (which == 1 ? Lq.b : Lq.r);
  const size_t pitch = sizeof(float) * Lp.H * Lp.W;
  SP_CUDA(cudaMemcpy2DAsync(rowp(dst, Lp, 0, r0), pitch, rowp(src, Lq, 0, r0), pitch,
                            sizeof(float) * (size_t)(r1 - r0) * Lp.W, g.C,
                            cudaMemcpyDeviceToDevice, s));
  return 0;
}

int stage_for(StripGroup& g, size_t bytes) {
  if (g.stage_bytes >= bytes) return 0;
  if (g.stage) cudaFreeHost(g.stage);
  g.stage = nullptr;
  g.stage_bytes = 0;
  SP_CUDA(cudaMallocHost(&g.stage, bytes));
  g.stage_bytes = bytes;
  return 0;
}

// host transport: rows [s0, s1) of every channel to strip q, rows [r0, r1)
// from it (pinned staging, stream-synchronous)
int host_sendrecv(StripGroup& g, float* buf, const Level& L, int q, int s0, int s1, int r0,
                  int r1, cudaStream_t s) {
  const size_t rowb = sizeof(float) * L.W, pitch = sizeof(float) * L.H * L.W;
  const size_t sb = (size_t)g.C * std::max(0, s1 - s0) * rowb;
  const size_t rb = (size_t)g.C * std::max(0, r1 - r0) * rowb;
  SP_TRY(stage_for(g, sb + rb + 16));
  char* sh = (char*)g.stage;
  char* rh = sh + sb;
  if (sb)
    SP_CUDA(cudaMemcpy2DAsync(sh, (s1 - s0) * rowb, rowp(buf, L, 0, s0), pitch, (s1 - s0) * rowb,
                              g.C, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  if (g.host.sendrecv(g.host.user, g.rank_of(q), sh, sb, rh, rb)) {
    set_error("host transport: send/recv with strip %d failed", q);
    return -1;
  }
  if (rb)
    SP_CUDA(cudaMemcpy2DAsync(rowp(buf, L, 0, r0), pitch, rh, (r1 - r0) * rowb, (r1 - r0) * rowb,
                              g.C, cudaMemcpyHostToDevice, s));
  SP_CUDA(cudaStreamSynchronize(s));
  return 0;
}

// halo exchange of buffer `which` (0 u, 1 b, 2 r) at partitioned level lv
int exchange(StripGroup& g, int lv, int which, cudaStream_t s) {
  if (g.P == 1) return 0;
  bool grouped = false;
  NcclApi* n = nccl();
  for (int i = 0; i < g.nloc; ++i) {
    const int p = g.first + i;
    const StripView& V = g.v[i][lv];
    Level& L = g.h[i]->lv[lv];
    void* buf = which == 0 ? L.u : (which == 1 ? L.b : L.r);
    // rows this strip needs: [e0, o0) from p-1 and [o1, e1) from p+1;
    // rows neighbours need from it: p-1 wants [o1(p-1), e1(p-1)), p+1 wants [e0(p+1), o0(p+1))
    for (int side = 0; side < 2; ++side) {
      const int q = side == 0 ? p - 1 : p + 1;
      if (q < 0 || q >= g.P) continue;
      const int rr0 = side == 0 ? V.e0 : V.o1, rr1 = side == 0 ? V.o0 : V.e1;
      if (g.local(q)) {
        SP_TRY(copy_rows(g, lv, which, p, q, rr0, rr1, s));
        continue;
      }
      // what q needs from p
      const int qo0 = g.o0[lv][q], qo1 = g.o1[lv][q];
      const int qe0 = std::max(0, qo0 - g.halo), qe1 = std::min(L.H, qo1 + g.halo);
      const int s0 = side == 0 ? qo1 : qe0, s1 = side == 0 ? qe1 : qo0;
      if (g.host_mode) {
        SP_TRY(host_sendrecv(g, (float*)buf, L, q, s0, s1, rr0, rr1, s));
        continue;
      }
      if (!g.comm || !n) { set_error("strip %d has no transport to strip %d", p, q); return -2; }
      if (!grouped) { SP_NCCL(n->GroupStart()); grouped = true; }
      for (int c = 0; c < g.C; ++c) {
        if (s1 > s0)
          SP_NCCL(n->Send(rowp(buf, L, c, s0), (size_t)(s1 - s0) * L.W, ncclFloat32, g.rank_of(q),
                          g.comm, s));
        if (rr1 > rr0)
          SP_NCCL(n->Recv(rowp(buf, L, c, rr0), (size_t)(rr1 - rr0) * L.W, ncclFloat32,
                          g.rank_of(q), g.comm, s));
      }
    }
  }
  if (grouped) SP_NCCL(n->GroupEnd());
  return 0;
}

// every strip's owned rows [o0, o1) of buffer `which` at level lv into every
// strip (used for the agglomerated level La and the final solution)
int gather_rows(StripGroup& g, int lv, int which, const std::vector<int>& r0,
                const std::vector<int>& r1, cudaStream_t s) {
  if (g.P == 1) return 0;
  NcclApi* n = nccl();
  for (int i = 0; i < g.nloc; ++i)
    for (int q = 0; q < g.P; ++q)
      if (q != g.first + i && g.local(q))
        SP_TRY(copy_rows(g, lv, which, g.first + i, q, r0[q], r1[q], s));
  if (g.nloc == g.P) return 0;
  Level& L = g.h[0]->lv[lv];
  void* buf = which == 0 ? L.u : (which == 1 ? L.b : L.r);
  if (g.host_mode) {
    // one strip per rank: broadcast every strip's owned rows from its rank
    const size_t rowb = sizeof(float) * L.W, pitch = sizeof(float) * L.H * L.W;
    for (int q = 0; q < g.P; ++q) {
      if (r1[q] <= r0[q]) continue;
      const size_t nb = (size_t)g.C * (r1[q] - r0[q]) * rowb;
      SP_TRY(stage_for(g, nb));
      const bool root = g.local(q);
      if (root)
        SP_CUDA(cudaMemcpy2DAsync(g.stage, (r1[q] - r0[q]) * rowb, rowp(buf, L, 0, r0[q]), pitch,
                                  (r1[q] - r0[q]) * rowb, g.C, cudaMemcpyDeviceToHost, s));
      SP_CUDA(cudaStreamSynchronize(s));
      if (g.host.bcast(g.host.user, g.stage, nb, g.rank_of(q))) {
        set_error("host transport: broadcast from strip %d failed", q);
        return -1;
      }
      if (!root)
        SP_CUDA(cudaMemcpy2DAsync(rowp(buf, L, 0, r0[q]), pitch, g.stage, (r1[q] - r0[q]) * rowb,
                                  (r1[q] - r0[q]) * rowb, g.C, cudaMemcpyHostToDevice, s));
      SP_CUDA(cudaStreamSynchronize(s));
    }
    return 0;
  }
  if (!g.comm || !n) { set_error("strip group spans ranks without a communicator"); return -2; }
  SP_NCCL(n->GroupStart());
  for (int q = 0; q < g.P; ++q)
    for (int c = 0; c < g.C; ++c)
      if (r1[q] > r0[q]) {
        float* p = rowp(buf, L, c, r0[q]);
        SP_NCCL(n->Broadcast(p, p, (size_t)(r1[q] - r0[q]) * L.W, ncclFloat32, g.rank_of(q),
                             g.comm, s));
      }
  SP_NCCL(n->GroupEnd());
  return 0;
}

// per-channel sum r^2 over the owned rows of every strip, bit-identical for
// every partition: residual on each view writing band partials, owned bands
// summed per strip, band sums combined across strips, total in band order
int residual_norms(StripGroup& g, int lv, bool exch, cudaStream_t s) {
  if (exch) SP_TRY(exchange(g, lv, 0, s));
  const int BR = march_band_rows();
  for (int i = 0; i < g.nloc; ++i) {
    const StripView& V = g.v[i][lv];
    Level& L = g.h[i]->lv[lv];
    const int hv = V.e1 - V.e0;
    const size_t ps = (size_t)L.H * L.W;
    if (tma_view_ok(L.W)) {
      // all channels in one launch: the view's planes keep the level's stride
      SP_TRY(resid_tma(rowp(L.u, L, 0, V.e0), rowp(L.b, L, 0, V.e0), mrow(L, V.e0),
                       rowp(L.r, L, 0, V.e0), nullptr, nullptr, nullptr, g.C, hv, L.W, s, 1,
                       nullptr, g.bandcol[i][lv], V.e0 / BR, g.nbt[lv], ps));
    } else {
      for (int c = 0; c < g.C; ++c)
        SP_TRY(resid_march(rowp(L.u, L, c, V.e0), rowp(L.b, L, c, V.e0), mrow(L, V.e0),
                           rowp(L.r, L, c, V.e0), nullptr, nullptr, nullptr, 1, hv, L.W, s, 1,
                           nullptr, g.bandcol[i][lv] + (size_t)c * g.nbt[lv] * g.ncg[lv],
                           V.e0 / BR, g.nbt[lv]));
    }
    const int n = g.C * g.nbt[lv];
    k_band_sum<<<cdiv(n, 256), 256, 0, s>>>(g.bandcol[i][lv], g.bands[i][lv], g.C, g.nbt[lv],
                                            g.ncg[lv], V.o0 / BR, cdiv(V.o1, BR));
    SP_CHECK_LAUNCH();
  }
  // combine: every band is owned by exactly one strip, the others hold +0
  if (g.P > 1) {
    for (int i = 0; i < g.nloc; ++i)
      for (int j = 0; j < g.nloc; ++j) {
        if (i == j) continue;
        const StripView& Vj = g.v[j][lv];
        const int b0 = Vj.o0 / BR, b1 = cdiv(Vj.o1, BR);
        SP_CUDA(cudaMemcpy2DAsync(g.bands[i][lv] + b0, sizeof(double) * g.nbt[lv],
                                  g.bands[j][lv] + b0, sizeof(double) * g.nbt[lv],
                                  sizeof(double) * (b1 - b0), g.C, cudaMemcpyDeviceToDevice, s));
      }
    if (g.nloc < g.P && g.host_mode) {
      const size_t nb = sizeof(double) * g.C * g.nbt[lv];
      SP_TRY(stage_for(g, nb));
      SP_CUDA(cudaMemcpyAsync(g.stage, g.bands[0][lv], nb, cudaMemcpyDeviceToHost, s));
      SP_CUDA(cudaStreamSynchronize(s));
      if (g.host.allreduce_f64(g.host.user, (double*)g.stage, (size_t)g.C * g.nbt[lv])) {
        set_error("host transport: all-reduce failed");
        return -1;
      }
      SP_CUDA(cudaMemcpyAsync(g.bands[0][lv], g.stage, nb, cudaMemcpyHostToDevice, s));
      SP_CUDA(cudaStreamSynchronize(s));
    } else if (g.nloc < g.P) {
      NcclApi* n = nccl();
      if (!g.comm || !n) { set_error("strip group spans ranks without a communicator"); return -2; }
      SP_NCCL(n->AllReduce(g.bands[0][lv], g.bands[0][lv], (size_t)g.C * g.nbt[lv],
                           ncclFloat64, ncclSum, g.comm, s));
    }
  }
  for (int i = 0; i < g.nloc; ++i) {
    k_band_total<<<1, 32, 0, s>>>(g.bands[i][lv], g.h[i]->lv[lv].norms, g.C, g.nbt[lv]);
    SP_CHECK_LAUNCH();
  }
  return 0;
}

// u (+)= P e on a view (coarse view from row e0 / 2, ch rows)
int prolong_view(StripGroup& g, Level& F, Level& G, const StripView& V, int ch, int hv,
                 int add, cudaStream_t s) {
  if (tma_prolong_ok(hv, F.W))
    return prolong_tma(rowp(G.u, G, 0, V.e0 / 2), rowp(F.u, F, 0, V.e0), rowp(F.b, F, 0, V.e0),
                       mrow(F, V.e0), g.C, ch, G.W, hv, F.W, add, s, 1, nullptr,
                       (size_t)F.H * F.W, (size_t)G.H * G.W);
  for (int c = 0; c < g.C; ++c)
    SP_TRY(prolong_march(rowp(G.u, G, c, V.e0 / 2), rowp(F.u, F, c, V.e0), rowp(F.b, F, c, V.e0),
                         mrow(F, V.e0), 1, ch, G.W, hv, F.W, add, s, 1, nullptr));
  return 0;
}

int oras_blend(StripGroup& g, int lv, cudaStream_t s) {
  for (int i = 0; i < g.nloc; ++i) {
    Hier* hh = g.h[i];
    const StripView& V = g.v[i][lv];
    Level& L = hh->lv[lv];
    const int hv = V.e1 - V.e0, npx = L.bh * L.bw, nb = L.nby * L.nbx;
    const size_t boff = (size_t)V.kya * L.nbx * npx, ps = (size_t)L.H * L.W;
    // all channels in one launch: corr channel planes keep the level's
    // block count (corr_nb), image planes the level's stride (ps)
    float* corr = (float*)L.corr + boff;
    SP_TRY(oras_local_launch<float>(rowp(L.r, L, 0, V.e0), mrow(L, V.e0), L.norms, L.tau_scale,
                                    V.ys, L.xs, V.nby, L.nbx, L.bh, L.bw, hv, L.W, g.C,
                                    hh->gamma, (long)npx, 1.0, (const float*)L.weights + boff,
                                    corr, s, 1, nullptr, 0, nb, ps,
                                    L.wdelta ? L.wdelta + (size_t)V.kya * L.nbx : nullptr));
    SP_TRY(oras_blend_launch<float>(rowp(L.u, L, 0, V.e0), corr, V.ys, L.xs, V.row_k0,
                                    V.row_n, L.col_k0, L.col_n, V.nby, L.nbx, L.bh, L.bw, hv,
                                    L.W, g.C, s, 1, nullptr, nb, ps));
  }
  return 0;
}

int smooth(StripGroup& g, int lv, int sweeps, bool first_done, cudaStream_t s) {
  for (int sw = 0; sw < sweeps; ++sw) {
    if (!(sw == 0 && first_done)) SP_TRY(residual_norms(g, lv, true, s));
    SP_TRY(oras_blend(g, lv, s));
  }
  return 0;
}

int vcycle(StripGroup& g, int lv, bool first_done, cudaStream_t s) {
  const HierCfg& cfg = g.h[0]->cfg;
  SP_TRY(smooth(g, lv, cfg.pre, first_done, s));
  const int nl = (int)g.h[0]->lv.size();
  if (lv + 1 >= nl) return 0;  // (La never includes the coarsest level)
  // residual + restriction on each view (correct on the owned coarse rows)
  for (int i = 0; i < g.nloc; ++i) {
    const StripView& V = g.v[i][lv];
    Level& F = g.h[i]->lv[lv];
    Level& G = g.h[i]->lv[lv + 1];
    if (tma_view_ok(F.W)) {
      SP_TRY(resid_restrict_tma(rowp(F.u, F, 0, V.e0), rowp(F.b, F, 0, V.e0), mrow(F, V.e0),
                                rowp(G.r, G, 0, V.e0 / 2), g.C, V.e1 - V.e0, F.W, s, 1, nullptr,
                                (size_t)F.H * F.W, (size_t)G.H * G.W));
    } else {
      for (int c = 0; c < g.C; ++c)
        SP_TRY(resid_restrict_march(rowp(F.u, F, c, V.e0), rowp(F.b, F, c, V.e0),
                                    mrow(F, V.e0), rowp(G.r, G, c, V.e0 / 2), 1, V.e1 - V.e0,
                                    F.W, s, 1, nullptr));
    }
  }
  if (lv + 1 < g.La) {
    SP_TRY(exchange(g, lv + 1, 2, s));
    for (int i = 0; i < g.nloc; ++i) {
      const StripView& V = g.v[i][lv + 1];
      Level& G = g.h[i]->lv[lv + 1];
      for (int c = 0; c < g.C; ++c)
        SP_TRY(sym_rhs<float>(rowp(G.r, G, c, V.e0), mrow(G, V.e0), rowp(G.b, G, c, V.e0),
                              rowp(G.u, G, c, V.e0), 1, V.e1 - V.e0, G.W, 1.0, s));
    }
    SP_TRY(vcycle(g, lv + 1, false, s));
  } else {
    // agglomerate: the owned coarse rows of every strip into every strip
    std::vector<int> r0(g.P), r1(g.P);
    for (int q = 0; q < g.P; ++q) {
      r0[q] = g.o0[lv][q] / 2;
      r1[q] = q == g.P - 1 ? g.h[0]->lv[lv + 1].H : g.o1[lv][q] / 2;
    }
    SP_TRY(gather_rows(g, lv + 1, 2, r0, r1, s));
    for (int i = 0; i < g.nloc; ++i) {
      Hier* hh = g.h[i];
      Level& G = hh->lv[lv + 1];
      SP_TRY(sym_rhs<float>((const float*)G.r, G.mask, (float*)G.b, (float*)G.u, g.C, G.H, G.W,
                            1.0, s, 1, hh->d_active));
      SP_TRY(vcycle_lv<float>(hh, lv + 1, false, s));
    }
  }
  // u += P e on each view (the coarse correction is valid around the owned rows)
  for (int i = 0; i < g.nloc; ++i) {
    const StripView& V = g.v[i][lv];
    Level& F = g.h[i]->lv[lv];
    Level& G = g.h[i]->lv[lv + 1];
    const int hv = V.e1 - V.e0, ch = std::min((hv + 1) / 2, G.H - V.e0 / 2);
    SP_TRY(prolong_view(g, F, G, V, ch, hv, 1, s));
  }
  SP_TRY(smooth(g, lv, cfg.post, false, s));
  return 0;
}

// FMG cascade (solver.py:302-317) with the partitioned levels on views
int cascade(StripGroup& g, cudaStream_t s) {
  const int nl = (int)g.h[0]->lv.size(), last = nl - 1;
  for (int i = 0; i < g.nloc; ++i) {
    Hier* hh = g.h[i];
    Level& Lc = hh->lv[last];
    SP_TRY(masked_sym_rhs<float>((const float*)Lc.values, Lc.mask, (float*)Lc.b, g.C, Lc.H,
                                 Lc.W, s, 1, hh->d_active));
    SP_TRY(enforce<float>((float*)Lc.u, (const float*)Lc.b, Lc.mask, g.C, Lc.H, Lc.W, 1, s, 1,
                          hh->d_active));
    SP_TRY(smooth_lv<float>(hh, last, 1, false, s));
    for (int lv = last - 1; lv >= g.La; --lv) {
      Level& F = hh->lv[lv];
      SP_TRY(masked_sym_rhs<float>((const float*)F.values, F.mask, (float*)F.b, g.C, F.H, F.W, s,
                                   1, hh->d_active));
      SP_TRY(prolong_lv<float>(hh, lv, 0, s));
      SP_TRY(smooth_lv<float>(hh, lv, 1, false, s));
    }
  }
  for (int lv = g.La - 1; lv >= 0; --lv) {
    for (int i = 0; i < g.nloc; ++i) {
      const StripView& V = g.v[i][lv];
      Level& F = g.h[i]->lv[lv];
      Level& G = g.h[i]->lv[lv + 1];
      const int hv = V.e1 - V.e0, ch = std::min((hv + 1) / 2, G.H - V.e0 / 2);
      for (int c = 0; c < g.C; ++c)
        SP_TRY(masked_sym_rhs<float>(rowp(F.values, F, c, V.e0), mrow(F, V.e0),
                                     rowp(F.b, F, c, V.e0), 1, hv, F.W, s));
      SP_TRY(prolong_view(g, F, G, V, ch, hv, 0, s));
    }
    SP_TRY(smooth(g, lv, 1, false, s));
  }
  return 0;
}

}  // namespace

// ---- C++ entry points (wrapped by capi) -------------------------------------------
int strip_create(StripGroup** out, int C, int H, int W, const HierCfg& cfg, int P, int nloc,
                 int first, int La, int halo, const int* o0, const int* o1, void* comm) {
  *out = nullptr;
  if (P < 1 || nloc < 1 || first < 0 || first + nloc > P || La < 0 || halo < 33 ||
      halo % march_band_rows()) {
    set_error("bad strip group (P %d, local %d from %d, La %d, halo %d)", P, nloc, first, La,
              halo);
    return -2;
  }
  // strips on other ranks need a transport: the NCCL communicator here, or a
  // host transport installed right after creation (sp_strip_set_host_transport);
  // an exchange without either fails with "no transport"
  if (tma_view_ok(128) && tma_prepare()) return -1;
  StripGroup* g = new StripGroup();
  g->P = P; g->nloc = nloc; g->first = first; g->La = La; g->halo = halo;
  g->C = C; g->H = H; g->W = W;
  g->comm = (ncclComm_t)comm;
  for (int i = 0; i < nloc; ++i) {
    Hier* h = nullptr;
    int rc = hier_create(&h, SP_F32, C, H, W, cfg, 1, 1);
    if (rc) { delete g; return rc; }
    h->use_graphs = false;
    g->h.push_back(h);
  }
  const int nl = (int)g->h[0]->lv.size();
  if (La > nl - 1) {
    set_error("%d partitioned levels but the hierarchy has %d (the coarsest is replicated)",
              La, nl);
    delete g;
    return -2;
  }
  const int BR = march_band_rows();
  g->o0.assign(La, std::vector<int>(P));
  g->o1.assign(La, std::vector<int>(P));
  g->v.assign(nloc, std::vector<StripView>(La));
  g->bandcol.assign(nloc, std::vector<double*>(La, nullptr));
  g->bands.assign(nloc, std::vector<double*>(La, nullptr));
  for (int lv = 0; lv < La; ++lv) {
    const Level& L = g->h[0]->lv[lv];
    if (L.W % 4 != 0 || L.W < 128) {  // row-marching sweeps (band-norm mode)
      set_error("partitioned level %d (%d x %d) needs W %% 4 == 0 and W >= 128", lv, L.H, L.W);
      delete g;
      return -2;
    }
    g->nbt.push_back(cdiv(L.H, BR));
    g->ncg.push_back(cdiv(L.W, 128));
    for (int p = 0; p < P; ++p) {
      g->o0[lv][p] = o0[(size_t)lv * P + p];
      g->o1[lv][p] = o1[(size_t)lv * P + p];
      const int a = g->o0[lv][p], b = g->o1[lv][p];
      const bool bad = a < 0 || b > L.H || b <= a || a % BR || (b % BR && b != L.H) ||
                       (p == 0 && a != 0) || (p == P - 1 && b != L.H) ||
                       (p > 0 && a != g->o1[lv][p - 1]) || (P > 1 && b - a < halo);
      if (bad) {
        set_error("strip %d rows [%d, %d) invalid at level %d (%d rows)", p, a, b, lv, L.H);
        delete g;
        return -2;
      }
    }
    for (int i = 0; i < nloc; ++i) {
      const int p = first + i;
      StripView V{};
      V.o0 = g->o0[lv][p];
      V.o1 = g->o1[lv][p];
      V.e0 = std::max(0, V.o0 - halo);
      V.e1 = std::min(L.H, V.o1 + halo);
      if (lv > 0 && V.e0 % 2) { set_error("odd view start"); delete g; return -2; }
      // block rows fully inside the view, their local starts and cover tables
      const int stride = cfg.block - cfg.overlap;
      std::vector<int> ysl;
      V.kya = -1;
      for (int k = 0; k < L.nby; ++k) {
        const int y0 = block_start(k, stride, L.H, L.bh);
        if (y0 >= V.e0 && y0 + L.bh <= V.e1) {
          if (V.kya < 0) V.kya = k;
          ysl.push_back(y0 - V.e0);
        }
      }
      V.nby = (int)ysl.size();
      const int hv = V.e1 - V.e0;
      std::vector<int> k0, n;
      cover_tables(ysl, L.bh, hv, k0, n);
      if (cudaMalloc((void**)&V.ys, sizeof(int) * std::max(1, V.nby)) != cudaSuccess ||
          cudaMalloc((void**)&V.row_k0, sizeof(int) * hv) != cudaSuccess ||
          cudaMalloc((void**)&V.row_n, sizeof(int) * hv) != cudaSuccess ||
          cudaMalloc((void**)&g->bandcol[i][lv],
                     sizeof(double) * C * g->nbt[lv] * g->ncg[lv]) != cudaSuccess ||
          cudaMalloc((void**)&g->bands[i][lv], sizeof(double) * C * g->nbt[lv]) != cudaSuccess) {
        set_error("strip table alloc failed");
        g->v[i][lv] = V;
        delete g;
        return -1;
      }
      g->v[i][lv] = V;
      if (V.nby < 1 ||
          cudaMemcpy(V.ys, ysl.data(), sizeof(int) * V.nby, cudaMemcpyHostToDevice) !=
              cudaSuccess ||
          cudaMemcpy(V.row_k0, k0.data(), sizeof(int) * hv, cudaMemcpyHostToDevice) !=
              cudaSuccess ||
          cudaMemcpy(V.row_n, n.data(), sizeof(int) * hv, cudaMemcpyHostToDevice) !=
              cudaSuccess) {
        set_error("strip view at level %d holds no whole block row", lv);
        delete g;
        return -2;
      }
    }
  }
  *out = g;
  return 0;
}

void strip_destroy(StripGroup* g) { delete g; }

int strip_set_host_transport(StripGroup* g, const HostTransport& t) {
  if (!t.sendrecv || !t.allreduce_f64 || !t.bcast) {
    set_error("host transport needs send/recv, all-reduce and broadcast callbacks");
    return -2;
  }
  if (g->graph) {
    cudaGraphExecDestroy(g->graph);
    g->graph = nullptr;
  }
  g->host = t;
  g->host_mode = true;
  return 0;
}

int strip_set_mask(StripGroup* g, const uint8_t* mask, const float* values, cudaStream_t s) {
  for (Hier* h : g->h) SP_TRY(hier_set_mask(h, mask, values, s));
  return 0;
}

// solver.py:328-372 on the strip group; bsym / u_io are full-size images
// (every rank holds the full right-hand side; u_io returns the gathered
// solution)
int strip_solve(StripGroup* g, const float* bsym, float* u_io, int init_mode, double tol,
                int cycles, int max_cycles, cudaStream_t s, SolveReport* rep) {
  // without partitioned levels every strip would run the same full solve
  if (g->La == 0)
    return hier_solve(g->h[0], bsym, u_io, init_mode, tol, cycles, max_cycles, s, nullptr,
                      nullptr, nullptr, rep);
  const int C = g->C;
  Level& L0 = g->h[0]->lv[0];
  const size_t n = (size_t)C * L0.H * L0.W;
  if (rep) { rep->iterations = 0; rep->nres = 0; rep->converged = 0; }
  SP_CUDA(cudaStreamSynchronize(s));
  for (Hier* h : g->h) {
    h->h_active[0] = 1;
    SP_CUDA(cudaMemcpyAsync(h->d_active, h->h_active, sizeof(int), cudaMemcpyHostToDevice, s));
  }
  if (init_mode == 2 && !g->h[0]->has_values) {
    set_error("hierarchy was built without stored values");
    return -2;
  }
  for (Hier* h : g->h) {
    Level& L = h->lv[0];
    if (init_mode == 1)
      SP_CUDA(cudaMemcpyAsync(L.u, u_io, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    else if (init_mode != 2)
      SP_CUDA(cudaMemsetAsync(L.u, 0, sizeof(float) * n, s));
  }
  // the cascade builds its own level right-hand sides (on views); the
  // solve's b~ goes in afterwards, as in solve_sym (solver.cu solve_t)
  if (init_mode == 2) SP_TRY(cascade(*g, s));
  for (Hier* h : g->h) {
    Level& L = h->lv[0];
    SP_CUDA(cudaMemcpyAsync(L.b, bsym, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    SP_TRY(enforce<float>((float*)L.u, (const float*)L.b, L.mask, C, L.H, L.W, 0, s));
  }
  int done = 0, cv = 0;
  auto norms0 = [&](bool exch) -> int { return residual_norms(*g, 0, exch, s); };
  auto cycle = [&]() -> int {
    if (g->host_mode) return vcycle(*g, 0, true, s);  // host callbacks: not capturable
    if (!g->graph) {
      if (!g->cap) SP_CUDA(cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking));
      // order the private capture stream after the work already queued on s
      cudaEvent_t ev;
      SP_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      SP_CUDA(cudaEventRecord(ev, s));
      SP_CUDA(cudaStreamWaitEvent(g->cap, ev, 0));
      SP_CUDA(cudaStreamSynchronize(g->cap));
      cudaEventDestroy(ev);
      cudaGraph_t gr;
      SP_CUDA(cudaStreamBeginCapture(g->cap, cudaStreamCaptureModeThreadLocal));
      int rc = vcycle(*g, 0, true, g->cap);
      cudaError_t e = cudaStreamEndCapture(g->cap, &gr);
      if (rc) { if (e == cudaSuccess) cudaGraphDestroy(gr); return rc; }
      SP_CUDA(e);
      size_t nn = 0;
      cudaGraphGetNodes(gr, nullptr, &nn);
      g->graph_nodes = (long long)nn;
      cudaError_t ie = cudaGraphInstantiate(&g->graph, gr, 0);
      cudaGraphDestroy(gr);
      SP_CUDA(ie);
    }
    SP_CUDA(cudaGraphLaunch(g->graph, s));
    count_launches(g->graph_nodes);
    return 0;
  };
  if (tol < 0) {
    for (int c = 0; c < cycles; ++c) {
      SP_TRY(norms0(true));
      SP_TRY(cycle());
    }
    done = cycles;
    cv = 1;
  } else {
    Hier* h0 = g->h[0];
    double* part = (double*)h0->d_scratch;
    double* bn = part + 1024;
    unsigned* counter = (unsigned*)(bn + 1);
    SP_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
    SP_TRY(chan_reduce<float>(0, (const float*)h0->lv[0].b, nullptr, nullptr, n, 1, part,
                              counter, bn, s));
    SP_CUDA(cudaMemcpyAsync(h0->h_norms, bn, sizeof(double), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    const double bnorm = std::sqrt(h0->h_norms[0]);
    const double scale = bnorm > 0 ? bnorm : 1.0;
    while (true) {
      SP_TRY(norms0(true));
      SP_CUDA(cudaMemcpyAsync(h0->h_norms, h0->lv[0].norms, sizeof(double) * C,
                              cudaMemcpyDeviceToHost, s));
      SP_CUDA(cudaStreamSynchronize(s));
      double tot = 0.0;
      for (int c = 0; c < C; ++c) tot += h0->h_norms[c];
      const double rel = std::sqrt(tot) / scale;
      if (rep && rep->nres < SP_MAX_RES) rep->residuals[rep->nres++] = rel;
      if (rel <= tol) { cv = 1; break; }
      if (done >= max_cycles) break;
      SP_TRY(cycle());
      ++done;
    }
  }
  if (rep) { rep->iterations = done; rep->converged = cv; }
  count_work(0, (long long)done * g->h[0]->lv[0].H * g->h[0]->lv[0].W);
  // gather the owned rows of the finest level into every strip
  std::vector<int> r0(g->P), r1(g->P);
  for (int q = 0; q < g->P; ++q) { r0[q] = g->o0[0][q]; r1[q] = g->o1[0][q]; }
  SP_TRY(gather_rows(*g, 0, 0, r0, r1, s));
  SP_CUDA(cudaMemcpyAsync(u_io, g->h[0]->lv[0].u, sizeof(float) * n, cudaMemcpyDeviceToDevice,
                          s));
  return 0;
}

int strip_levels(StripGroup* g, int* nlev, int* dims, int cap) {
  Hier* h = g->h[0];
  *nlev = (int)h->lv.size();
  for (int i = 0; i < *nlev && 2 * i + 1 < cap; ++i) {
    dims[2 * i] = h->lv[i].H;
    dims[2 * i + 1] = h->lv[i].W;
  }
  return 0;
}

}  // namespace sp
