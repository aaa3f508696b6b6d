/*
 * dos.h — C ABI of libdos.so, the B200-native Deep Optimizer States update
 * phase (arXiv 2410.21316).  Plain pointers and sizes only; no torch types.
 *
 * Every entry point returns 0 on success or a negative DOS_E* code; the
 * message for the calling thread is available from dos_last_error().
 * Error classes mirror the reference's exception types:
 *   DOS_EINVAL -> ValueError, DOS_ETYPE -> TypeError, DOS_ECUDA/DOS_ESYS ->
 *   RuntimeError, DOS_EINFEASIBLE -> InfeasibleConfigError.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/optistate):
 *   dos_adam_step_host / dos_adam_step_cuda
 *       kernels.py:107-139 adam_step_arrays (validation + scalars in Python,
 *       the per-element loop here), kernels.py:88-101 _adam_step_jit,
 *       fused with core.py:201-205 upscale (grad load) and
 *       core.py:190-198 downscale_rne (working-copy store).
 *   dos_downscale_host / dos_upscale_host / dos_downscale_cuda / dos_upscale_cuda
 *       core.py:190-198 downscale_rne, core.py:201-205 upscale,
 *       executor.py:317-349 flush_gradients (GPU_UPSCALE_FP32 leg).
 *   dos_host_alloc / dos_host_free
 *       core.py:208-272 ShardedOptimizer's flat arrays -> a pinned host pool.
 *   dos_exec_* (the copy-stream / host-lane engine)
 *       executor.py:174-235 ExecutorTarget.apply (numeric effect per action)
 *       driven by scheduler.py:402-466 run_update (one submit per action, in
 *       emission order); executor.py:120-171 EmulatedDevice -> HBM slots.
 */
#ifndef DOS_H
#define DOS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define DOS_OK 0
#define DOS_EINVAL (-1)
#define DOS_ETYPE (-2)
#define DOS_ECUDA (-3)
#define DOS_ESYS (-4)
#define DOS_EINFEASIBLE (-5)
#define DOS_ESTATE (-6) /* structural violation (double stage, missing triplet, ...) */

/* element dtypes */
#define DOS_NONE (-1)
#define DOS_F32 0
#define DOS_F16 1
#define DOS_BF16 2

/* Per-step scalars, prepared by the caller exactly as kernels.py:122-135:
 * bc1/bc2 = f32(1 - pow(beta, step)) in double, lr/betas/eps cast to f32.
 * (1 - beta) is formed on the device/host as the fp32 difference 1.0f - beta.
 * adamw != 0 applies decoupled weight decay p = p * (1 - lr*wd) before the
 * Adam step (no reference pin: the reference has no weight decay). */
typedef struct dos_adam_scalars {
  float lr, beta1, beta2, eps, bc1, bc2, weight_decay;
  int32_t adamw;
} dos_adam_scalars;

const char* dos_last_error(void);
int dos_version(void);
/* Number of libdos kernels launched by this process so far (K1 + conversions). */
int64_t dos_launch_count(void);

/* ---- K1: fused Adam on the GPU (sm_100a).  Asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default).  p/m/v fp32 in place; g in
 * g_dtype (F32/F16/BF16); if lowp_dtype != DOS_NONE the updated params are
 * also written to p_lowp in that dtype (RNE) in the same pass. */
int dos_adam_step_cuda(float* p, float* m, float* v, const void* g, int g_dtype,
                       void* p_lowp, int lowp_dtype, int64_t n,
                       const dos_adam_scalars* s, void* stream);

/* K1 with the all-gather fused into its epilogue: as dos_adam_step_cuda,
 * and every updated half-precision element is also stored to peer_lowp[r]
 * (r < npeers <= DOS_MAX_PEERS), e.g. NVLink-mapped peer buffers.
 * Replaces executor.py:219-227 FLUSH_OUT_MODEL16 + the ZeRO-3 param
 * all-gather; requires lowp_dtype != DOS_NONE. */
int dos_adam_step_cuda_bcast(float* p, float* m, float* v, const void* g, int g_dtype,
                             void* p_lowp, int lowp_dtype, void* const* peer_lowp, int npeers,
                             int64_t n, const dos_adam_scalars* s, void* stream);

/* K1 with the reduce-scatter fused into its grad load (and, optionally, the
 * all-gather into its epilogue): g_src[r] (r < nsrc <= DOS_MAX_PEERS + 1, in
 * rank order) holds rank r's grads for this range; g_src[self] is local and
 * streamed by TMA, the others are loaded over NVLink one tile ahead.  The
 * grads used are lowp(rank-order fp32 sum) [then lowp(x * grad_scale) if
 * grad_scale != 1]; 16-bit grads only, working copy in the same dtype.
 * Replaces the bucketed NCCL reduce-scatter before the phase. */
int dos_adam_step_cuda_rs(float* p, float* m, float* v, const void* const* g_src, int nsrc, int self,
                          int g_dtype, float grad_scale, void* p_lowp, int lowp_dtype,
                          void* const* peer_lowp, int npeers, int64_t n, const dos_adam_scalars* s,
                          void* stream);

/* Stand-alone reduce-scatter of one range with the same rounding:
 * out[i] = lowp(sum_r src[r][i]) (scaled as above); out may alias a source
 * (in place).  Used for the host subgroups' grads before their D2H flush. */
int dos_reduce_scatter_cuda(void* out, const void* const* src, int nsrc, int dtype, float scale,
                            int64_t n, void* stream);

/* ---- Post-phase coherence (executor.py:271-282: model16 == downscale_rne(params32)
 * for every subgroup, asserted after each phase).  Each range compares
 * lowp[i] with RNE(p32[i]) in `nwin` windows of `window` elements: the whole
 * range when nwin*window >= n, else windows spread evenly from its first
 * element to its last (a sample).  p32/lowp may be HBM or registered pinned
 * host memory.  Asynchronous on `stream`; out (device, 2 x u64, caller
 * initialises to {0, ~0}) receives the mismatch count and the smallest
 * (range_index << 40 | element) key. */
typedef struct dos_coh_range {
  const float* p32;
  const void* lowp;
  int64_t n, window, nwin;
} dos_coh_range;
int dos_coherence_cuda(const dos_coh_range* ranges, int nranges, int lowp_dtype,
                       unsigned long long* out, void* stream);

/* ---- CUDA IPC for symmetric full-model buffers (one process per GPU).
 * export: the handle of the allocation containing dev_ptr and dev_ptr's
 * byte offset in it; import: map a peer's allocation (cached) and return
 * base + offset; close: unmap everything this process imported. */
int dos_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset);
int dos_ipc_import(const unsigned char handle[64], uint64_t offset, void** dev_ptr);
int dos_ipc_close_all(void);

/* ---- H1: the same update on host cores (bit-identical results).  Blocks
 * the calling thread only; nthreads <= 0 uses the library's host team. */
int dos_adam_step_host(float* p, float* m, float* v, const void* g, int g_dtype,
                       void* p_lowp, int lowp_dtype, int64_t n,
                       const dos_adam_scalars* s, int nthreads);

/* ---- conversions (numpy-exact fp16 incl. NaN payloads; torch-exact bf16) */
int dos_downscale_host(const float* x, void* out, int out_dtype, int64_t n, int nthreads);
int dos_upscale_host(const void* x, int in_dtype, float* out, int64_t n, int nthreads);
int dos_downscale_cuda(const float* x, void* out, int out_dtype, int64_t n, void* stream);
int dos_upscale_cuda(const void* x, int in_dtype, float* out, int64_t n, void* stream);

/* ---- host pool: page-aligned, THP-advised, first-touched by the host
 * team, then page-locked and registered with CUDA (if a device is present
 * and register_cuda != 0).  numa_node < 0: no binding. */
int dos_host_alloc(size_t bytes, int numa_node, int register_cuda, void** out);
int dos_host_free(void* ptr);
/* Sparse pool regions: reserve address space for a whole flat array, commit
 * (first touch + page-lock + register) only the byte ranges homed on the
 * host.  Committed runs that touch are merged into one registration.
 * dos_host_committed returns the committed bytes (or a negative DOS_E*).
 * dos_host_free releases either kind.  Replaces core.py:208-272's dense
 * allocation of every array for the whole shard: subgroups whose fp32 state
 * is homed in HBM cost no host memory. */
int dos_host_reserve(size_t bytes, int numa_node, int register_cuda, void** out);
int dos_host_commit(void* base, size_t offset, size_t len);
int64_t dos_host_committed(void* base);
int dos_host_threads(void); /* size of the library's host team */
/* Host memory probe (the host-DRAM roofline's denominator): one pass of the
 * team over `bytes`, reading src (mode 0) or copying src -> dst (mode 1);
 * the pass's wall seconds in *seconds.  Not on the update path. */
int dos_host_membw(const void* src, void* dst, size_t bytes, int mode, int nthreads, double* seconds);
int dos_set_host_threads(int n);

/* ---- the copy-stream / host-lane engine ---------------------------------
 * Action kinds and lanes use the reference's enum order
 * (scheduler.py:43-89). */
enum dos_action_kind {
  DOS_CPU_UPDATE = 0,
  DOS_GPU_UPDATE = 1,
  DOS_CPU_DOWNSCALE = 2,
  DOS_H2D_PARAMS16 = 3,
  DOS_FLUSH_OUT_MODEL16 = 4,
  DOS_FLUSH_OUT_M = 5,
  DOS_FLUSH_OUT_V = 6,
  DOS_FLUSH_OUT_P = 7,
  DOS_PREFETCH_M = 8,
  DOS_PREFETCH_V = 9,
  DOS_PREFETCH_P = 10,
  DOS_GRAD_FLUSH = 11
};
enum dos_lane { DOS_LANE_CPU = 0, DOS_LANE_FAST = 1, DOS_LANE_H2D = 2, DOS_LANE_D2H = 3 };

/* Where one rank's state lives.  Host arrays are indexed by the flat shard
 * offset; device static-resident state is compact (static_offset[i] gives the
 * element offset of subgroup i in dev_static_{p,m,v}, -1 if not static). */
typedef struct dos_state_desc {
  int32_t num_subgroups;
  const int64_t* sg_start; /* [num_subgroups] */
  const int64_t* sg_size;  /* [num_subgroups] */
  const int64_t* static_offset; /* [num_subgroups], -1 = not resident */
  int32_t lowp_dtype;      /* DOS_F16 or DOS_BF16: grads and working copy */
  /* host (pinned) */
  float* host_p;
  float* host_m;
  float* host_v;
  const void* host_g;      /* lowp grads for CPU subgroups (flushed before the phase) */
  void* host_lowp;         /* staging for CPU-downscaled params (H2D_PARAMS16 source) */
  /* device (HBM) */
  const void* dev_g;       /* lowp grads, whole shard */
  void* dev_lowp;          /* working copy, whole shard */
  float* dev_static_p;
  float* dev_static_m;
  float* dev_static_v;
  /* host_io != 0: the step's grads arrive in host_g for every subgroup and
   * the working copy must also land in host_lowp.  Fast subgroups then copy
   * their grads H2D inside PREFETCH_P (static: inside GPU_UPDATE, before K1)
   * and their working copy D2H inside FLUSH_OUT_P (static: inside
   * FLUSH_OUT_MODEL16), so the extra 2+2 B/param ride the same lanes. */
  int32_t host_io;
  /* Fused all-gather of the working copy (ZeRO-3, one node).  peer_lowp[r]
   * is where THIS rank's shard starts inside peer r's full-model buffer
   * (an IPC-mapped NVLink address, see dos_ipc_*).  K1 stores each updated
   * half-precision element to the local working copy and to every peer in
   * the same pass; a host subgroup's working copy is forwarded peer-to-peer
   * by the copy engine right after its H2D_PARAMS16.  npeers <= DOS_MAX_PEERS. */
  int32_t npeers;
  void* const* peer_lowp;
  /* flush_grads != 0: the gradient flush of SURVEY §8(f) row 1 runs inside
   * the phase — each CPU_UPDATE's bf16/fp16 grads are copied dev_g -> host_g
   * (pinned DMA, in subgroup order, on a dedicated stream) and the host lane
   * waits only for its own subgroup's copy; the upcast is fused into H1. */
  int32_t flush_grads;
  /* Fused reduce-scatter of the grads (ZeRO-3, one node), replacing the
   * bucketed NCCL reduce-scatter before the phase.  nsrc_g = world size
   * (0 = off); src_g[r] is where THIS rank's shard starts inside rank r's
   * full-model grad buffer (r in rank order; src_g[self_rank] must be
   * dev_g — peers are IPC-mapped NVLink addresses).  A subgroup's grads are
   * lowp(fp32 sum over r in rank order), then lowp(that * grad_scale) when
   * grad_scale != 1.  GPU_UPDATE reduces inside K1 (peer loads over NVLink);
   * a CPU_UPDATE's grads are reduced into dev_g on the grad stream right
   * before their in-phase flush, so nsrc_g > 0 requires flush_grads and
   * excludes host_io.  Every rank must have finished writing its grads before
   * the phase starts, and none may overwrite them until every rank's phase
   * has ended (the caller's barriers). */
  int32_t nsrc_g;
  int32_t self_rank;
  const void* const* src_g;
  float grad_scale;
  /* Optional per-subgroup HBM homes of the static residents' fp32 state:
   * dev_static_sg[3*i + {0,1,2}] = p, m, v of subgroup i (NULL when not
   * static).  When non-NULL it replaces dev_static_{p,m,v} + static_offset[i]
   * (static_offset[i] >= 0 still marks residency), so the static set can
   * grow and shrink one subgroup at a time without re-packing HBM. */
  float* const* dev_static_sg;
  /* host_io only: 0 ships every static resident's grads H2D at phase start
   * (best when the residents' updates come last); k > 0 issues each
   * resident's grads when its GPU_UPDATE is submitted, k resident updates
   * ahead of the fast lane, so the copy engine interleaves them with the
   * H2D lane instead of draining them all first (best when they lead). */
  int32_t host_io_ahead;
  /* How many CPU_UPDATE actions the plan holds (-1: unknown).  0 lets the
   * engine skip the host lane's staging-ring shuttle for this phase (plans
   * with no host-updated subgroup keep every SM for K1). */
  int32_t host_updates;
} dos_state_desc;

#define DOS_MAX_PEERS 7

typedef struct dos_exec_config {
  int32_t device;
  int32_t num_slots;      /* physical HBM windows (1 or 2) */
  int64_t slot_elems;     /* elements per slot piece (>= largest dynamic subgroup) */
  int32_t host_threads;   /* <=0: library default team */
  int32_t fuse_downscale; /* !=0: CPU_UPDATE writes host_lowp; CPU_DOWNSCALE is a marker */
} dos_exec_config;

typedef struct dos_action_desc {
  int32_t id;
  int32_t kind;
  int32_t subgroup;     /* -1 for batched CPU_DOWNSCALE */
  int32_t lane;
  int32_t is_static;    /* the subgroup is fast-tier resident */
  int32_t num_deps;
  const int32_t* deps;
  int32_t batch_len;
  const int32_t* batch;
} dos_action_desc;

int dos_exec_create(const dos_exec_config* cfg, void** out);
int dos_exec_destroy(void* ex);
/* Start a phase: binds state + scalars, records the t0 marker.  max_actions
 * bounds the action ids of this phase. */
int dos_exec_begin(void* ex, const dos_state_desc* st, const dos_adam_scalars* s,
                   int32_t max_actions);
/* Enqueue one action (never waits on the GPU or the host lane). */
int dos_exec_submit(void* ex, const dos_action_desc* a);
/* Wait for the phase; fills measured [start,end) in ns since t0 per action id
 * (arrays of length >= number of submitted actions). */
int dos_exec_finish(void* ex, int64_t* start_ns, int64_t* end_ns, int32_t n);
/* Make `stream` (a cudaStream_t) wait until submitted device action `id` of
 * the current phase has finished — e.g. start the all-gather of a subgroup's
 * working copy as soon as its GPU_UPDATE / H2D_PARAMS16 is done, while the
 * rest of the phase still runs.  Host-lane actions are rejected (EINVAL). */
int dos_exec_stream_wait(void* ex, int32_t id, void* stream);
/* Device pointer of a staging slot piece (0=m,1=v,2=p) for tests/inspection. */
int dos_exec_slot_ptr(void* ex, int32_t slot, int32_t piece, float** out);

#ifdef __cplusplus
}
#endif
#endif /* DOS_H */
