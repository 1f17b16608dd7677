// solver.cuh -- device-resident multigrid hierarchy (see solver.cu).
#pragma once
#include <algorithm>
#include <vector>

#include "kernels.cuh"

#define SP_MAX_RES 256

namespace sp {

// host-staged strip transport (strips.cu): caller callbacks over pinned
// host buffers; each returns 0 on success
struct HostTransport {
  int (*sendrecv)(void* user, int peer, const void* send, size_t send_bytes, void* recv,
                  size_t recv_bytes) = nullptr;
  int (*allreduce_f64)(void* user, double* buf, size_t n) = nullptr;
  int (*bcast)(void* user, void* buf, size_t bytes, int root) = nullptr;
  void* user = nullptr;
};

struct HierCfg {
  int block = 32, overlap = 6, levels = 0, pre = 1, post = 1;
  double alpha = 1.0, rho = 0.25;
};

struct Level {
  int H, W, bh, bw, nby, nbx;
  double tau_scale;
  uint8_t* mask;
  void *values, *u, *b, *r, *corr, *weights;
  double* partial;
  size_t npart;
  unsigned* counter;
  double* norms;
  int *ys, *xs, *row_k0, *row_n, *col_k0, *col_n;
  int* wdelta;  // [nby * nbx] shared-weight aliases (float levels), or null
  // [ntile][nby * nbx][32] ORAS job row masks (float levels, blocks <= 32 x
  // 32): bit s of word j = row s of column j is masked or outside the block;
  // rebuilt with the mask pyramid (set_mask_t), or null
  uint32_t* offbits;
  int *rowinfo, *colinfo;  // packed cover words (oras.cu blend_pack), or null
  bool pair_cols;  // W even and every block column start even (k_oras_blend3q)
};

struct Hier {
  int dtype = 0, C = 1, ntile = 1;
  HierCfg cfg;
  double gamma = 0.0;
  bool has_values = false;
  bool use_graphs = true;
  int sweep = 2;               // 2 TMA, 1 row-marching, 0 per-pixel (solver.cu)
  std::vector<Level> lv;
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  long long graph_nodes = 0;
  double* h_norms = nullptr;   // pinned [ntile][C]
  int* h_active = nullptr;     // pinned [ntile]
  int* d_active = nullptr;     // [ntile] read by every V-cycle kernel
  void* d_scratch = nullptr;   // reduction partials
  // channel-parallel V-cycle (solver.cu run_vcycle): C non-owning one-channel
  // views of this hierarchy and the streams their graph branches run on
  bool owner = true;
  cudaEvent_t up_ev = nullptr;  // recorded after each h_active upload
  // device-driven tolerance loop (solver.cu solve_loop_t): one graph launch
  // per solve, a WHILE conditional node around {stop test; IF{V-cycle;
  // residual}}; loop_ctl holds the test's inputs and the iteration record
  cudaGraphExec_t loop_exec = nullptr;
  void* loop_ctl = nullptr;
  void* h_loop = nullptr;       // pinned copy of loop_ctl (read back once)
  long long loop_nodes = 0;
  // compacted active-tile list of the fused tile solves (tilesolve.cu)
  int* d_list = nullptr;
  int* h_list = nullptr;       // pinned
  cudaEvent_t list_ev = nullptr;
  std::vector<Hier*> chv;
  std::vector<cudaStream_t> ch_streams;
  std::vector<cudaEvent_t> ch_events;
  ~Hier();
};

// C-layout report (mirrors include/sparsepaint_b200.h sp_solve_report)
struct SolveReport {
  int iterations;
  int converged;
  int nres;
  int pad;
  double residuals[SP_MAX_RES];
};

int hier_create(Hier** out, int dtype, int C, int H, int W, const HierCfg& cfg,
                int with_values, int ntile = 1);
int hier_set_mask(Hier* h, const uint8_t* mask, const void* values, cudaStream_t s);
// u_in (optional): the start iterate for init_mode 1 (default: u_io itself);
// src_mode 1: `bsym` holds stored values x and b~ = C~ (mask ? x : 0) is
// formed directly in the hierarchy's level-0 right-hand side
int hier_solve(Hier* h, const void* bsym, void* u_io, int init_mode, double tol,
               int cycles, int max_cycles, cudaStream_t s, const int* active_in, int* iters,
               int* conv, SolveReport* rep, const void* u_in = nullptr, int src_mode = 0);
int hier_vcycle(Hier* h, const void* bsym, void* u_io, cudaStream_t s);
// h_active (pinned) may be rewritten once the last upload from it is done
int active_host_ready(Hier* h);
int upload_active(Hier* h, cudaStream_t s);

// tilesolve.cu: fused on-chip cold solve of a batch of small tiles
bool tile_fused_ok(const Hier* h);
int tile_solve_fused(Hier* h, const float* bsym, float* u_out, double tol, int max_cycles,
                     cudaStream_t s, const int* active_in, int* iters, int* conv);

// level operations (solver.cu), used by the row-strip solver (strips.cu)
template <typename T>
int prolong_lv(Hier* h, int lv, int add, cudaStream_t s);
template <typename T>
int smooth_lv(Hier* h, int lv, int sweeps, bool first_done, cudaStream_t s);
template <typename T>
int vcycle_lv(Hier* h, int lv, bool first_done, cudaStream_t s);

// vec.cu: deterministic reductions (fixed CTA count per size)
size_t red_partials();  // doubles needed in `partial` per reduced channel
template <typename T>
int dot_self(const T* x, size_t n, double* partial, unsigned* counter, double* out,
             cudaStream_t s);

}  // namespace sp
