// dos_exec.cpp — the copy-stream / host-lane engine of the update phase.
//
// The reference executes a plan by calling ExecutorTarget.apply once per
// action in emission order from one thread (scheduler.py:402-466 run_update,
// executor.py:192-235 apply), with numpy copies standing in for the fast
// tier (executor.py:120-171 EmulatedDevice).  Here each submit() *enqueues*
// the action's real effect and returns immediately:
//
//   lane FAST_COMPUTE -> CUDA stream `fast`  (K1; FLUSH_OUT_MODEL16 is fused
//                                             into K1's working-copy store)
//   lane H2D          -> CUDA stream `h2d`   (pinned cudaMemcpyAsync)
//   lane D2H          -> CUDA stream `d2h`   (pinned cudaMemcpyAsync)
//   lane CPU_COMPUTE  -> one host worker thread driving the H1 team
//
// Each lane is FIFO in emission order, exactly the reference's lane model.
// Dependencies: GPU->GPU by cudaStreamWaitEvent; host->GPU by
// cuStreamWaitValue32 on a per-action flag in mapped pinned memory (the host
// worker writes the phase epoch when the action ends), so the dispatcher
// never blocks; GPU->host by cudaEventSynchronize in the worker.  Emission
// order is topological and every lane serves it in order, so no wait can
// deadlock.
//
// Staging (Alg. 1's p_tmp/m_tmp/v_tmp): `num_slots` HBM
// windows of {m, v, p}.  A window is taken at PREFETCH_M and released by the
// last of its flushes; a new window waits for that flush's end event.  This
// physically double-buffers what the reference models as one staging buffer
// per state stream, so the next subgroup's prefetch overlaps the current
// update and flush (the plan itself is unchanged).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dos_internal.h"

namespace {

typedef CUresult (*pfn_wait_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*pfn_write_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// Working-copy staging rings of the host lane (dos_host_adam_ring + the
// shuttle kernel): per team thread `slots` x `chunk` elements of pinned
// memory, meant to stay in the host's caches so the working copy of a
// host-updated subgroup never makes a DRAM round trip.  OFF by default
// (DOS_W_RING=1 turns it on): measured on the 16-core B200 host it is slower
// than H1 storing the working copy non-temporally into the host image and
// H2D_PARAMS16 shipping it (1035-1122 ms vs 976-997 ms for the 7B phase,
// profiles/r02_ring_ab.jsonl) — the slots' regular stores pay a
// read-for-ownership after every device read, as cached stores into the
// image do (1092-1126 ms), and the zero-copy pull shares the link with the
// copy engines (profiles/r02_zero_copy_pull.json).
struct RingCfg {
  bool on;
  int slots;      // per team thread
  int64_t chunk;  // elements per slot
  int ctas;       // shuttle CTAs
};
// Grad ring of the in-phase flush (dos_gring): `slots` rows of `chunk`
// elements per team thread.  OFF by default (DOS_G_RING=1 turns it on):
// measured on the 16-core B200 host it is slower than the whole-subgroup D2H
// into the host image (7B phase 1167-1354 ms vs 974-1022 ms,
// profiles/r02_gring_ab.jsonl): the row copies share the copy engines with
// the streamed windows' 400 MB flushes, so a row the team waits for can sit
// behind one for milliseconds, and a ring small enough to stay in the LLC
// has well under a millisecond of slack.
struct GRingCfg {
  bool on;
  int slots;
  int64_t chunk;
};
const GRingCfg& gring_cfg() {
  static GRingCfg c = [] {
    GRingCfg r{false, 3, 1 << 16};  // 3 rows x 16 threads x 64K elements = 6 MB of bf16
    if (const char* e = getenv("DOS_G_RING")) r.on = strcmp(e, "0") != 0;
    if (const char* e = getenv("DOS_G_RING_SLOTS")) r.slots = std::max(1, std::min(64, atoi(e)));
    if (const char* e = getenv("DOS_G_RING_CHUNK")) r.chunk = std::max<int64_t>(1024, atoll(e)) & ~int64_t(63);
    return r;
  }();
  return c;
}

// Split copies (A/B knob, off by default): each H2D-lane copy of a subgroup
// (PREFETCH_M/V/P, H2D_PARAMS16) — and with DOS_D2H_SPLIT each FLUSH_OUT_* —
// goes out as k pieces on k streams (the lane's own + k-1 helpers forked and
// joined by events), so more copy engines keep host reads in flight while the
// host team loads the DRAM.  The action still ends when its last piece has.
int split_env(const char* name) {
  const char* e = getenv(name);
  return e ? std::max(1, std::min(8, atoi(e))) : 1;
}
int h2d_split() {
  static const int k = split_env("DOS_H2D_SPLIT");
  return k;
}
int d2h_split() {
  static const int k = split_env("DOS_D2H_SPLIT");
  return k;
}

const RingCfg& ring_cfg() {
  static RingCfg c = [] {
    RingCfg r{false, 4, 1 << 16, 16};  // per thread 4 x 64K elements (512 KB of bf16: the core's L2)
    if (const char* e = getenv("DOS_W_RING")) r.on = strcmp(e, "0") != 0;
    if (const char* e = getenv("DOS_W_RING_SLOTS")) r.slots = std::max(1, std::min(64, atoi(e)));
    if (const char* e = getenv("DOS_W_RING_CHUNK")) r.chunk = std::max<int64_t>(1024, atoll(e)) & ~int64_t(63);
    if (const char* e = getenv("DOS_SHUTTLE_CTAS")) r.ctas = std::max(1, std::min(32, atoi(e)));
    return r;
  }();
  return c;
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

#define DOS_CU(call)                                                                                       \
  do {                                                                                                     \
    cudaError_t e__ = (call);                                                                              \
    if (e__ != cudaSuccess) return dos_set_error(DOS_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e__)); \
  } while (0)

enum { PIECE_M = 0, PIECE_V = 1, PIECE_P = 2 };

struct Job {
  int32_t id, kind, sg;
  std::vector<int32_t> deps, batch;
  cudaEvent_t flushed = nullptr;  // in-phase grad flush of this subgroup (flush_grads)
  bool gring = false;             // grads arrive row by row through the grad ring
  uint32_t gseq0 = 0;             // its first row's sequence number
};

struct Engine {
  int dev = 0;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // fast, h2d, d2h
  cudaStream_t gst = nullptr;                        // in-phase grad flush (D2H); host_io: residents' grads H2D
  cudaStream_t ost = nullptr;                        // host_io: residents' working copy D2H
  cudaStream_t pst = nullptr;                        // fused all-gather: host subgroups' peer forwards
  cudaStream_t hst[2][7] = {};                       // split-copy helpers of the h2d / d2h lanes
  cudaEvent_t sev_fork[2] = {}, sev_join[2][7] = {};
  cudaStream_t wst = nullptr;                        // the shuttle kernel's stream
  // staging ring (see RingCfg) served by the shuttle kernel; ring_phase: used in this phase
  bool ring_phase = false;
  uint16_t* ring_mem = nullptr;
  uint16_t* ring_mem_dev = nullptr;                   // its device alias (the shuttle reads it over PCIe)
  int ring_threads = 0;                               // team threads the slots are laid out for
  std::vector<int64_t> ring_last;                     // per thread slot: its last shuttle descriptor (-1: none)
  int64_t ring_sg_start = 0;                          // subgroup being shipped
  uint32_t* ring_flags = nullptr;                     // mapped: per subgroup, epoch once its last chunk landed
  CUdeviceptr ring_flags_dev = 0;
  int32_t ring_flags_cap = 0;
  pfn_write_value32 write_fn = nullptr;
  // grad ring (GRingCfg): pinned rows + mapped ready/consumed flags
  bool gring_phase = false;
  int gring_k = 0;                  // slice layout's thread count
  uint16_t* gring_mem = nullptr;
  size_t gring_bytes = 0;
  uint32_t* gring_flags = nullptr;  // [0, slots): ready; [slots, 2 slots): consumed
  CUdeviceptr gring_flags_dev = 0;
  std::vector<int> gring_counts;
  uint32_t gring_seq = 0;           // rows issued so far (monotonic across phases)
  // the shuttle: descriptor queue in mapped pinned memory
  dos_shuttle_ctl* sh_ctl = nullptr;
  dos_shuttle_ctl* sh_ctl_dev = nullptr;
  std::atomic<uint32_t> sh_next{0};  // next descriptor number (monotonic across phases; posted by many threads)
  uint32_t sh_phase_first = 0;       // first descriptor number of the running shuttle
  bool sh_running = false;
  std::vector<cudaEvent_t> ev_g;                      // per action: its grads are on the host
  std::vector<cudaEvent_t> ev_sg;                     // per subgroup: host_io grads of a static resident landed
  std::deque<int32_t> static_q;                       // host_io_ahead: resident updates whose grads are in flight
  static constexpr int kFlushAhead = 4;               // flush_grads: host updates a grad flush may run ahead
  std::deque<int32_t> flush_q;                        // flush_grads: host updates whose grads were flushed
  int nslots = 0;
  int64_t slot_elems = 0;
  float* slot_mem = nullptr;
  bool fuse = true;
  int host_threads = 0;

  // phase
  bool active = false;
  dos_state_desc S{};
  std::vector<int64_t> sg_start, sg_size, static_off;
  dos_kscal K{};
  dos_peers peers{0, {}};  // fused all-gather targets (shard element 0 in each peer)
  dos_gsrc gsrc{0, 0, 1.0f, {}};  // fused reduce-scatter sources (shard element 0 in each rank)
  int32_t max_actions = 0, count = 0;
  std::vector<cudaEvent_t> ev_s, ev_e;
  cudaEvent_t ev0 = nullptr;
  std::vector<uint8_t> is_host;
  std::vector<int64_t> host_s, host_e;
  uint32_t* flags = nullptr;  // mapped pinned
  CUdeviceptr flags_dev = 0;
  int32_t flags_cap = 0;
  uint32_t epoch = 0;
  pfn_wait_value32 wait_fn = nullptr;
  bool wait_value_ok = true;
  int64_t host_t0 = 0;

  // staging bookkeeping
  std::vector<int> sg_slot;
  std::vector<uint8_t> sg_mask;
  int next_slot = 0;
  int slot_release[2] = {-1, -1};  // action id whose end frees the slot; -2 = window open
  int slot_owner[2] = {-1, -1};

  // dispatcher error (first one wins)
  int err = DOS_OK;
  std::string errmsg;

  // host lane
  std::thread worker;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::deque<Job> q;
  bool stop = false;
  int inflight = 0;
  std::vector<uint8_t> host_done;
  int host_err = DOS_OK;
  std::string host_errmsg;

  float* slot_ptr(int s, int piece) { return slot_mem + ((int64_t)s * 3 + piece) * slot_elems; }

  int fail(int code, const std::string& msg) {
    if (err == DOS_OK) {
      err = code;
      errmsg = msg;
    }
    return dos_set_error(code, "%s", msg.c_str());
  }

  // ---- host worker
  void worker_loop() {
    cudaSetDevice(dev);
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || !q.empty(); });
        if (q.empty()) return;
        j = std::move(q.front());
        q.pop_front();
      }
      int rc = DOS_OK;
      std::string msg;
      for (int32_t d : j.deps) {
        if (!is_host[d]) {
          cudaError_t e = cudaEventSynchronize(ev_e[d]);
          if (e != cudaSuccess && rc == DOS_OK) {
            rc = DOS_ECUDA;
            msg = std::string("waiting on GPU dep failed: ") + cudaGetErrorString(e);
          }
        }
      }
      if (j.flushed) {  // this subgroup's grads reached the host image
        cudaError_t e = cudaEventSynchronize(j.flushed);
        if (e != cudaSuccess && rc == DOS_OK) {
          rc = DOS_ECUDA;
          msg = std::string("waiting on the grad flush failed: ") + cudaGetErrorString(e);
        }
      }
      const int64_t t_s = now_ns();
      if (rc == DOS_OK) rc = run_host(j, msg);
      const int64_t t_e = now_ns();
      {
        std::lock_guard<std::mutex> lk(mu);
        host_s[j.id] = t_s - host_t0;
        host_e[j.id] = t_e - host_t0;
        host_done[j.id] = 1;
        if (rc != DOS_OK && host_err == DOS_OK) {
          host_err = rc;
          host_errmsg = msg;
        }
        --inflight;
      }
      __atomic_store_n(&flags[j.id], epoch, __ATOMIC_RELEASE);
      done_cv.notify_all();
    }
  }

  // ---- shuttle queue (host side; only the host worker posts)
  static void spin_pause(int i) {
    if (i < 512) __builtin_ia32_pause();
    else std::this_thread::yield();
  }
  bool sh_done(uint32_t id) const {
    const uint32_t d = __atomic_load_n(&sh_ctl->done[id % DOS_SHUTTLE_Q], __ATOMIC_ACQUIRE);
    return (int32_t)(d - (id + 1)) >= 0;
  }
  int sh_wait(uint32_t id) {
    for (int i = 0; !sh_done(id); ++i) {
      spin_pause(i);
      if ((i & 0xFFFF) == 0xFFFF) {  // a dead shuttle must not hang the host lane
        const cudaError_t q = cudaStreamQuery(wst);
        if (q == cudaSuccess) return dos_set_error(DOS_ESTATE, "shuttle exited before descriptor %u", id);
        if (q != cudaErrorNotReady) return dos_set_error(DOS_ECUDA, "shuttle failed: %s", cudaGetErrorString(q));
      }
    }
    return DOS_OK;
  }
  // any team thread may post (the queue is multi-producer: numbers are
  // claimed atomically, each descriptor is published by its own id store)
  int64_t sh_post(const void* src_dev, void* dst_dev, uint32_t bytes, int32_t flag_idx, uint32_t flag_val) {
    const uint32_t id = sh_next.fetch_add(1, std::memory_order_relaxed);
    // the queue slot's previous descriptor (same phase) must be done
    if (id - sh_phase_first >= DOS_SHUTTLE_Q) {
      const int rc = sh_wait(id - DOS_SHUTTLE_Q);
      if (rc != DOS_OK) return rc;
    }
    dos_shuttle_desc& d = sh_ctl->q[id % DOS_SHUTTLE_Q];
    d.src = (uint64_t)(uintptr_t)src_dev;
    d.dst = (uint64_t)(uintptr_t)dst_dev;
    d.bytes = bytes;
    d.flag_idx = flag_idx;
    d.flag_val = flag_val;
    __atomic_store_n(&d.id, id + 1, __ATOMIC_RELEASE);  // publishes the fields (x86: store order)
    return id;
  }

  // staging-ring callbacks (run on every team thread)
  static int64_t ring_post(void* ctx, const uint16_t* slot, int64_t off, int64_t cnt) {
    Engine* e = static_cast<Engine*>(ctx);
    char* dst = static_cast<char*>(e->S.dev_lowp) + 2 * (e->ring_sg_start + off);
    return e->sh_post(e->ring_mem_dev + (slot - e->ring_mem), dst, (uint32_t)(2 * cnt), -1, 0);
  }
  static int ring_wait(void* ctx, int64_t id) { return static_cast<Engine*>(ctx)->sh_wait((uint32_t)id); }

  // the shuttle runs for the whole phase: stop it once everything is posted
  void sh_stop() {
    if (!sh_running) return;
    __atomic_store_n(&sh_ctl->stop, 1u, __ATOMIC_RELEASE);
    sh_running = false;
  }

  int run_host(const Job& j, std::string& msg) {
    const int lt = S.lowp_dtype;
    if (j.kind == DOS_CPU_UPDATE && ring_phase) {
      // the working copy leaves through the team's LLC-resident staging
      // slots, served by the shuttle; once every chunk has landed the
      // subgroup's flag releases its H2D_PARAMS16
      const int64_t a = sg_start[j.sg], n = sg_size[j.sg];
      const RingCfg& rc = ring_cfg();
      std::fill(ring_last.begin(), ring_last.end(), -1);
      dos_ring r{ring_mem, ring_threads, rc.slots, rc.chunk, this, ring_post, ring_wait};
      ring_sg_start = a;
      int code = dos_host_adam_ring(S.host_p + a, S.host_m + a, S.host_v + a,
                                    static_cast<const char*>(S.host_g) + 2 * a, lt, lt, n, K, host_threads, r,
                                    ring_last.data());
      for (int64_t id : ring_last)
        if (code == DOS_OK && id >= 0) code = sh_wait((uint32_t)id);
      if (code == DOS_OK) __atomic_store_n(&ring_flags[j.sg], epoch, __ATOMIC_RELEASE);
      if (code != DOS_OK) msg = dos_last_error();
      return code;
    }
    if (j.kind == DOS_CPU_UPDATE && j.gring) {
      const int64_t a = sg_start[j.sg], n = sg_size[j.sg];
      const GRingCfg& gc = gring_cfg();
      dos_gring r{gring_mem, gc.slots, gc.chunk, gring_k, gring_flags, gring_flags + gc.slots, gring_counts.data(),
                  j.gseq0};
      void* lp = fuse ? static_cast<void*>(static_cast<char*>(S.host_lowp) + 2 * a) : nullptr;
      const int rc = dos_host_adam_gring(S.host_p + a, S.host_m + a, S.host_v + a, lt, lp, lt, n, K, r);
      if (rc != DOS_OK) msg = dos_last_error();
      return rc;
    }
    if (j.kind == DOS_CPU_UPDATE) {
      const int64_t a = sg_start[j.sg], n = sg_size[j.sg];
      const void* g = static_cast<const char*>(S.host_g) + 2 * a;
      void* lp = fuse ? static_cast<void*>(static_cast<char*>(S.host_lowp) + 2 * a) : nullptr;
      const int rc = dos_host_adam(S.host_p + a, S.host_m + a, S.host_v + a, g, lt, lp, fuse ? lt : DOS_NONE, n, K,
                                   host_threads);
      if (rc != DOS_OK) msg = dos_last_error();
      return rc;
    }
    if (j.kind == DOS_CPU_DOWNSCALE) {
      if (fuse) return DOS_OK;  // already written by the fused CPU_UPDATE
      for (int32_t b : j.batch) {
        const int64_t a = sg_start[b], n = sg_size[b];
        const int rc = dos_host_down(S.host_p + a, static_cast<char*>(S.host_lowp) + 2 * a, lt, n, host_threads);
        if (rc != DOS_OK) {
          msg = dos_last_error();
          return rc;
        }
      }
      return DOS_OK;
    }
    msg = "action kind " + std::to_string(j.kind) + " is not a host-lane action";
    return DOS_EINVAL;
  }

  void wait_host_action(int32_t id) {
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return host_done[id] != 0; });
  }

  // ---- GPU dependency edges
  int gpu_wait_deps(cudaStream_t s, const dos_action_desc* a) {
    for (int k = 0; k < a->num_deps; ++k) {
      const int32_t d = a->deps[k];
      if (is_host[d]) {
        bool done = false;
        if (wait_value_ok && wait_fn) {
          CUresult r = wait_fn((CUstream)s, flags_dev + 4 * (CUdeviceptr)d, epoch, CU_STREAM_WAIT_VALUE_GEQ);
          if (r == CUDA_SUCCESS) done = true;
          else wait_value_ok = false;  // fall back to blocking the dispatcher
        }
        if (!done) wait_host_action(d);
      } else {
        DOS_CU(cudaStreamWaitEvent(s, ev_e[d], 0));
      }
    }
    return DOS_OK;
  }

  int submit(const dos_action_desc* a) {
    if (!active) return fail(DOS_ESTATE, "dos_exec_submit outside a phase");
    if (a->id != count || a->id >= max_actions)
      return fail(DOS_EINVAL, "action id " + std::to_string(a->id) + " out of emission order (expected " +
                                  std::to_string(count) + ")");
    for (int k = 0; k < a->num_deps; ++k)
      if (a->deps[k] < 0 || a->deps[k] >= a->id)
        return fail(DOS_EINVAL, "action " + std::to_string(a->id) + " has a forward dependency");
    const int sg = a->subgroup;
    if (a->kind != DOS_CPU_DOWNSCALE && (sg < 0 || sg >= S.num_subgroups))
      return fail(DOS_EINVAL, "action " + std::to_string(a->id) + " names subgroup " + std::to_string(sg));
    ++count;

    if (a->lane == DOS_LANE_CPU) {
      is_host[a->id] = 1;
      Job j;
      j.id = a->id;
      j.kind = a->kind;
      j.sg = sg;
      j.deps.assign(a->deps, a->deps + a->num_deps);
      j.batch.assign(a->batch, a->batch + a->batch_len);
      for (int32_t b : j.batch)
        if (b < 0 || b >= S.num_subgroups) return fail(DOS_EINVAL, "downscale batch names a bad subgroup");
      if (S.flush_grads && a->kind == DOS_CPU_UPDATE && gring_phase) {
        // the grads of this subgroup D2H row by row through the grad ring,
        // every copy enqueued now (FIFO-safe: each waits only for rows the
        // host consumes before it needs this subgroup)
        const int64_t start = sg_start[sg], n = sg_size[sg];
        if (gsrc.n > 0) {  // fused reduce-scatter of this subgroup, in place in dev_g, ahead of its rows
          const int rc = dos_reduce_launch(static_cast<char*>(const_cast<void*>(S.dev_g)) + 2 * start, S.lowp_dtype, n,
                                           dos_gsrc_offset(gsrc, start), gst);
          if (rc != DOS_OK) return fail(rc, dos_last_error());
        }
        const int rc = enqueue_grad_rows(start, n, &j.gseq0);
        if (rc != DOS_OK) return fail(rc, dos_last_error());
        j.gring = true;
      } else if (S.flush_grads && a->kind == DOS_CPU_UPDATE) {
        // §8(f) row 1 inside the phase: this subgroup's half-precision grads
        // D2H on their own stream, in emission (= subgroup) order
        const int64_t start = sg_start[sg], n = sg_size[sg];
        // Throttle: this subgroup's flush is issued once the host lane has
        // finished the CPU update kFlushAhead positions earlier, so the grads
        // still land well before H1 needs them but the D2H copy engine is not
        // monopolised by every host subgroup's grads at phase start (the
        // streamed windows' FLUSH_OUT_* share it).
        if ((int)flush_q.size() >= kFlushAhead) {
          const int32_t d = flush_q.front();
          flush_q.pop_front();
          if (wait_value_ok && wait_fn &&
              wait_fn((CUstream)gst, flags_dev + 4 * (CUdeviceptr)d, epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            wait_value_ok = false;
        }
        flush_q.push_back(a->id);
        if (gsrc.n > 0) {  // fused reduce-scatter of this subgroup, in place in dev_g, then the flush
          const int rc = dos_reduce_launch(static_cast<char*>(const_cast<void*>(S.dev_g)) + 2 * start, S.lowp_dtype, n,
                                           dos_gsrc_offset(gsrc, start), gst);
          if (rc != DOS_OK) return fail(rc, dos_last_error());
        }
        DOS_CU(cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(S.host_g)) + 2 * start,
                               static_cast<const char*>(S.dev_g) + 2 * start, (size_t)n * 2, cudaMemcpyDeviceToHost,
                               gst));
        DOS_CU(cudaEventRecord(ev_g[a->id], gst));
        j.flushed = ev_g[a->id];
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        q.push_back(std::move(j));
        ++inflight;
      }
      cv.notify_one();
      return DOS_OK;
    }

    cudaStream_t s = a->lane == DOS_LANE_FAST ? st[0] : a->lane == DOS_LANE_H2D ? st[1] : st[2];
    int rc = gpu_wait_deps(s, a);
    if (rc == DOS_OK && a->kind == DOS_PREFETCH_M && !a->is_static && sg_slot[sg] < 0) rc = open_window(sg, s);
    if (rc != DOS_OK) return fail(rc, dos_last_error());
    DOS_CU(cudaEventRecord(ev_s[a->id], s));
    rc = enqueue_gpu(a, s);
    if (rc != DOS_OK) return fail(rc, dos_last_error());
    DOS_CU(cudaEventRecord(ev_e[a->id], s));
    return DOS_OK;
  }

  // The grad ring's D2H rows of one subgroup on the grad stream.
  int enqueue_grad_rows(int64_t start, int64_t n, uint32_t* seq0) {
    const GRingCfg& gc = gring_cfg();
    const int k = gring_k;
    const int64_t C = gc.chunk, per = dos_gring_per(n, k), rows = n > 0 ? dos_gring_rows(n, k, C) : 0;
    const uint32_t R = (uint32_t)gc.slots;
    *seq0 = gring_seq;
    const char* dev_g = static_cast<const char*>(S.dev_g) + 2 * start;
    for (int64_t c = 0; c < rows; ++c) {
      const uint32_t seq = gring_seq++;
      const uint32_t slot = seq % R;
      char* dst = reinterpret_cast<char*>(gring_mem) + (size_t)slot * k * C * 2;
      if (seq >= R &&  // the slot's previous row must have been consumed by every thread
          wait_fn((CUstream)gst, gring_flags_dev + 4 * (CUdeviceptr)(R + slot), seq - R + 1, CU_STREAM_WAIT_VALUE_GEQ) !=
              CUDA_SUCCESS)
        return dos_set_error(DOS_ECUDA, "cuStreamWaitValue32 (grad ring) failed");
      bool full = true;
      for (int t = 0; t < k && full; ++t) {
        const int64_t lo = std::min(n, per * t), hi = std::min(n, lo + per);
        if (lo + c * C < hi && lo + (c + 1) * C > hi) full = false;
        if (lo + c * C >= hi) full = false;
      }
      if (full) {
        DOS_CU(cudaMemcpy2DAsync(dst, (size_t)C * 2, dev_g + 2 * c * C, (size_t)per * 2, (size_t)C * 2, (size_t)k,
                                 cudaMemcpyDeviceToHost, gst));
      } else {
        for (int t = 0; t < k; ++t) {
          const int64_t lo = std::min(n, per * t), hi = std::min(n, lo + per), c0 = lo + c * C;
          if (c0 >= hi) continue;
          DOS_CU(cudaMemcpyAsync(dst + (size_t)t * C * 2, dev_g + 2 * c0, (size_t)std::min(C, hi - c0) * 2,
                                 cudaMemcpyDeviceToHost, gst));
        }
      }
      if (write_fn((CUstream)gst, gring_flags_dev + 4 * (CUdeviceptr)slot, seq + 1, 0) != CUDA_SUCCESS)
        return dos_set_error(DOS_ECUDA, "cuStreamWriteValue32 (grad ring) failed");
    }
    return DOS_OK;
  }

  // A window opens at PREFETCH_M: take the next physical slot and make the
  // stream wait for the flush that released it (before the start stamp).
  int open_window(int sg, cudaStream_t s) {
    const int sl = next_slot;
    if (slot_release[sl] == -2)
      return dos_set_error(DOS_EINFEASIBLE, "subgroup %d opens a window while slot %d (subgroup %d) is still unflushed",
                           sg, sl, slot_owner[sl]);
    if ((int64_t)sg_size[sg] > slot_elems)
      return dos_set_error(DOS_EINFEASIBLE, "subgroup %d (%lld) exceeds the HBM window", sg, (long long)sg_size[sg]);
    if (slot_release[sl] >= 0) DOS_CU(cudaStreamWaitEvent(s, ev_e[slot_release[sl]], 0));
    next_slot = (sl + 1) % nslots;
    slot_release[sl] = -2;
    slot_owner[sl] = sg;
    sg_slot[sg] = sl;
    return DOS_OK;
  }

  // host_io transfers (see dos_state_desc.host_io)
  cudaError_t copy_grads_h2d(int64_t start, int64_t n, cudaStream_t s) {
    return cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(S.dev_g)) + 2 * start,
                           static_cast<const char*>(S.host_g) + 2 * start, (size_t)n * 2, cudaMemcpyHostToDevice, s);
  }
  cudaError_t copy_lowp_d2h(int64_t start, int64_t n, cudaStream_t s) {
    return cudaMemcpyAsync(static_cast<char*>(S.host_lowp) + 2 * start, static_cast<const char*>(S.dev_lowp) + 2 * start,
                           (size_t)n * 2, cudaMemcpyDeviceToHost, s);
  }

  // One lane copy as k pieces on the lane stream + k-1 helpers (see h2d_split).
  int lane_copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    const int dir = kind == cudaMemcpyHostToDevice ? 0 : 1;
    const int k = dir == 0 ? h2d_split() : d2h_split();
    const size_t piece = ((bytes + k - 1) / k + 4095) & ~size_t(4095);
    if (k == 1 || bytes < 2 * piece) {
      DOS_CU(cudaMemcpyAsync(dst, src, bytes, kind, s));
      return DOS_OK;
    }
    if (!sev_fork[dir]) {
      DOS_CU(cudaEventCreateWithFlags(&sev_fork[dir], cudaEventDisableTiming));
      for (int h = 0; h < 7; ++h) {
        DOS_CU(cudaStreamCreateWithFlags(&hst[dir][h], cudaStreamNonBlocking));
        DOS_CU(cudaEventCreateWithFlags(&sev_join[dir][h], cudaEventDisableTiming));
      }
    }
    DOS_CU(cudaEventRecord(sev_fork[dir], s));
    int h = 0;
    for (size_t off = piece; off < bytes; off += piece, ++h) {
      const size_t n = std::min(piece, bytes - off);
      DOS_CU(cudaStreamWaitEvent(hst[dir][h], sev_fork[dir], 0));
      DOS_CU(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n, kind,
                             hst[dir][h]));
      DOS_CU(cudaEventRecord(sev_join[dir][h], hst[dir][h]));
    }
    DOS_CU(cudaMemcpyAsync(dst, src, std::min(piece, bytes), kind, s));
    for (int i = 0; i < h; ++i) DOS_CU(cudaStreamWaitEvent(s, sev_join[dir][i], 0));
    return DOS_OK;
  }

  int enqueue_gpu(const dos_action_desc* a, cudaStream_t s) {
    const int sg = a->subgroup;
    const int64_t start = sg_start[sg], n = sg_size[sg];
    const int lt = S.lowp_dtype;
    char* dev_lowp = static_cast<char*>(S.dev_lowp);
    const char* dev_g = static_cast<const char*>(S.dev_g);
    switch (a->kind) {
      case DOS_PREFETCH_M:
      case DOS_PREFETCH_V:
      case DOS_PREFETCH_P: {
        if (a->is_static) return dos_set_error(DOS_ESTATE, "static subgroup %d prefetched", sg);
        const int piece = a->kind == DOS_PREFETCH_M ? PIECE_M : a->kind == DOS_PREFETCH_V ? PIECE_V : PIECE_P;
        if (n > slot_elems) return dos_set_error(DOS_EINFEASIBLE, "subgroup %d (%lld) exceeds the HBM window", sg, (long long)n);
        if (sg_slot[sg] < 0) return dos_set_error(DOS_ESTATE, "subgroup %d prefetched before its window opened", sg);
        if (sg_mask[sg] & (1u << piece))
          return dos_set_error(DOS_ESTATE, "subgroup %d piece %c staged twice", sg, "mvp"[piece]);
        sg_mask[sg] |= (uint8_t)(1u << piece);
        const float* src = (piece == PIECE_M ? S.host_m : piece == PIECE_V ? S.host_v : S.host_p) + start;
        if (const int rc = lane_copy(slot_ptr(sg_slot[sg], piece), src, (size_t)n * 4, cudaMemcpyHostToDevice, s))
          return rc;
        if (S.host_io && piece == PIECE_P) DOS_CU(copy_grads_h2d(start, n, s));
        return DOS_OK;
      }
      case DOS_GPU_UPDATE: {
        const void* g = dev_g + 2 * start;
        void* lp = dev_lowp + 2 * start;
        if (a->is_static) {
          const int64_t o = static_off[sg];
          if (o < 0) return dos_set_error(DOS_ESTATE, "subgroup %d marked static but has no HBM residence", sg);
          if (S.host_io) {
            if (S.host_io_ahead > 0) {
              // ship this resident's grads now, at most host_io_ahead resident
              // updates ahead of the fast lane
              if ((int)static_q.size() >= S.host_io_ahead) {
                DOS_CU(cudaStreamWaitEvent(gst, ev_s[static_q.front()], 0));
                static_q.pop_front();
              }
              DOS_CU(copy_grads_h2d(start, n, gst));
              DOS_CU(cudaEventRecord(ev_sg[sg], gst));
              static_q.push_back(a->id);
            }
            // (host_io_ahead == 0: shipped H2D at phase start on the side stream)
            DOS_CU(cudaStreamWaitEvent(s, ev_sg[sg], 0));
          }
          float* sp = S.dev_static_sg ? S.dev_static_sg[3 * sg] : S.dev_static_p + o;
          float* sm = S.dev_static_sg ? S.dev_static_sg[3 * sg + 1] : S.dev_static_m + o;
          float* sv = S.dev_static_sg ? S.dev_static_sg[3 * sg + 2] : S.dev_static_v + o;
          if (!sp || !sm || !sv) return dos_set_error(DOS_ESTATE, "static subgroup %d has no HBM state", sg);
          return dos_adam_launch(sp, sm, sv, g, lt, lp, lt, n, K, s, dos_peers_offset(peers, start),
                                 dos_gsrc_offset(gsrc, start));
        }
        if (sg_slot[sg] < 0 || sg_mask[sg] != 7u)
          return dos_set_error(DOS_ESTATE, "fast update of subgroup %d with missing pieces (mask %u)", sg,
                               (unsigned)sg_mask[sg]);
        const int sl = sg_slot[sg];
        return dos_adam_launch(slot_ptr(sl, PIECE_P), slot_ptr(sl, PIECE_M), slot_ptr(sl, PIECE_V), g, lt, lp, lt, n,
                               K, s, dos_peers_offset(peers, start), dos_gsrc_offset(gsrc, start));
      }
      case DOS_FLUSH_OUT_MODEL16:
        // K1 already stored the working copy in the same pass.
        if (!a->is_static && !(sg_slot[sg] >= 0 && (sg_mask[sg] & (1u << PIECE_P))))
          return dos_set_error(DOS_ESTATE, "FLUSH_OUT_MODEL16 of subgroup %d without staged params", sg);
        if (S.host_io && a->is_static) {
          // mirror a resident's working copy on its own side stream, off the
          // compute lane and not queued behind the residents' grads H2D (gst)
          DOS_CU(cudaEventRecord(ev_sg[sg], s));
          DOS_CU(cudaStreamWaitEvent(ost, ev_sg[sg], 0));
          DOS_CU(copy_lowp_d2h(start, n, ost));
        }
        return DOS_OK;
      case DOS_FLUSH_OUT_M:
      case DOS_FLUSH_OUT_V:
      case DOS_FLUSH_OUT_P: {
        const int piece = a->kind == DOS_FLUSH_OUT_M ? PIECE_M : a->kind == DOS_FLUSH_OUT_V ? PIECE_V : PIECE_P;
        if (sg_slot[sg] < 0 || !(sg_mask[sg] & (1u << piece)))
          return dos_set_error(DOS_ESTATE, "subgroup %d piece %c not resident on device", sg, "mvp"[piece]);
        float* dst = (piece == PIECE_M ? S.host_m : piece == PIECE_V ? S.host_v : S.host_p) + start;
        const int sl = sg_slot[sg];
        if (const int rc = lane_copy(dst, slot_ptr(sl, piece), (size_t)n * 4, cudaMemcpyDeviceToHost, s)) return rc;
        if (S.host_io && piece == PIECE_P) DOS_CU(copy_lowp_d2h(start, n, s));
        sg_mask[sg] &= (uint8_t)~(1u << piece);
        if (sg_mask[sg] == 0) {  // window closes with this flush
          slot_release[sl] = a->id;
          sg_slot[sg] = -1;
        }
        return DOS_OK;
      }
      case DOS_H2D_PARAMS16:
        if (ring_phase) {
          // the chunks already went H2D through the staging ring during the
          // CPU update: wait until its last one has landed
          if (wait_fn((CUstream)s, ring_flags_dev + 4 * (CUdeviceptr)sg, epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return dos_set_error(DOS_ECUDA, "cuStreamWaitValue32 (staging ring) failed");
        } else {
          if (const int rc = lane_copy(dev_lowp + 2 * start, static_cast<const char*>(S.host_lowp) + 2 * start,
                                       (size_t)n * 2, cudaMemcpyHostToDevice, s))
            return rc;
        }
        // fused all-gather for a host subgroup: forward it peer-to-peer (NVLink
        // copy engines) on the peer stream, chained by event, so the next
        // subgroup's prefetches on the H2D lane do not queue behind N-1 copies
        if (peers.n > 0) {
          DOS_CU(cudaEventRecord(ev_g[a->id], s));
          DOS_CU(cudaStreamWaitEvent(pst, ev_g[a->id], 0));
          for (int r = 0; r < peers.n; ++r)
            DOS_CU(cudaMemcpyAsync(peers.p[r] + start, dev_lowp + 2 * start, (size_t)n * 2, cudaMemcpyDeviceToDevice,
                                   pst));
        }
        return DOS_OK;
      default:
        return dos_set_error(DOS_EINVAL, "unexpected action kind %d on a device lane", a->kind);
    }
  }

  int begin(const dos_state_desc* st_desc, const dos_adam_scalars* sc, int32_t nmax) {
    if (active) return dos_set_error(DOS_ESTATE, "a phase is already active");
    if (!st_desc || !sc) return dos_set_error(DOS_EINVAL, "NULL state or scalars");
    if (st_desc->lowp_dtype != DOS_F16 && st_desc->lowp_dtype != DOS_BF16)
      return dos_set_error(DOS_ETYPE, "working-copy dtype %d unsupported", st_desc->lowp_dtype);
    if (nmax < 0) return dos_set_error(DOS_EINVAL, "max_actions must be >= 0");
    DOS_CU(cudaSetDevice(dev));
    if (sh_running) {  // a shuttle left over by a begin() that failed after launching it
      sh_stop();
      cudaStreamSynchronize(wst);
      dos_reserve_sms(0);
    }
    S = *st_desc;
    const int ns = S.num_subgroups;
    sg_start.assign(S.sg_start, S.sg_start + ns);
    sg_size.assign(S.sg_size, S.sg_size + ns);
    if (S.static_offset) static_off.assign(S.static_offset, S.static_offset + ns);
    else static_off.assign(ns, -1);
    K = dos_make_kscal(sc);
    if (S.npeers < 0 || S.npeers > DOS_MAX_PEERS || (S.npeers > 0 && !S.peer_lowp))
      return dos_set_error(DOS_EINVAL, "npeers must be in [0, %d] with peer pointers", DOS_MAX_PEERS);
    peers.n = S.npeers;
    for (int r = 0; r < S.npeers; ++r) peers.p[r] = static_cast<uint16_t*>(S.peer_lowp[r]);
    gsrc = dos_gsrc{0, 0, 1.0f, {}};
    if (S.nsrc_g != 0) {
      if (S.nsrc_g < 1 || S.nsrc_g > DOS_MAX_PEERS + 1 || !S.src_g)
        return dos_set_error(DOS_EINVAL, "nsrc_g must be in [1, %d] with source pointers", DOS_MAX_PEERS + 1);
      if (S.self_rank < 0 || S.self_rank >= S.nsrc_g || S.src_g[S.self_rank] != S.dev_g)
        return dos_set_error(DOS_EINVAL, "src_g[self_rank] must be this rank's dev_g");
      if (!S.flush_grads || S.host_io)
        return dos_set_error(DOS_EINVAL, "the fused reduce-scatter needs flush_grads and excludes host_io");
      if (!(S.grad_scale > 0.0f)) return dos_set_error(DOS_EINVAL, "grad_scale must be positive");
      gsrc.n = S.nsrc_g;
      gsrc.self = S.self_rank;
      gsrc.scale = S.grad_scale;
      for (int r = 0; r < S.nsrc_g; ++r) {
        if (!S.src_g[r]) return dos_set_error(DOS_EINVAL, "NULL grad source %d", r);
        gsrc.p[r] = static_cast<const uint16_t*>(S.src_g[r]);
      }
    }
    const int32_t cap = nmax > 0 ? nmax : 1;
    while ((int32_t)ev_s.size() < cap) {
      cudaEvent_t a, b, c;
      DOS_CU(cudaEventCreate(&a));
      DOS_CU(cudaEventCreate(&b));
      DOS_CU(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
      ev_s.push_back(a);
      ev_e.push_back(b);
      ev_g.push_back(c);
    }
    if (flags_cap < cap) {
      if (flags) cudaFreeHost(flags);
      flags = nullptr;
      int32_t want = std::max(cap, 1024);
      DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&flags), (size_t)want * 4, cudaHostAllocMapped));
      memset(flags, 0, (size_t)want * 4);
      void* dptr = nullptr;
      DOS_CU(cudaHostGetDevicePointer(&dptr, flags, 0));
      flags_dev = (CUdeviceptr)dptr;
      flags_cap = want;
      epoch = 0;
    }
    if (ring_flags_cap < ns) {
      if (ring_flags) cudaFreeHost(ring_flags);
      ring_flags = nullptr;
      const int32_t want = std::max(ns, 256);
      DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&ring_flags), (size_t)want * 4, cudaHostAllocMapped));
      memset(ring_flags, 0, (size_t)want * 4);
      void* dptr = nullptr;
      DOS_CU(cudaHostGetDevicePointer(&dptr, ring_flags, 0));
      ring_flags_dev = (CUdeviceptr)dptr;
      ring_flags_cap = want;
      // flags written in earlier epochs must not satisfy this phase's waits
      memset(flags, 0, (size_t)flags_cap * 4);
      epoch = 0;
    }
    ++epoch;
    if (epoch == 0) {  // wrapped: reset
      memset(flags, 0, (size_t)flags_cap * 4);
      memset(ring_flags, 0, (size_t)ring_flags_cap * 4);
      epoch = 1;
    }
    // the staging ring carries the working copy of host-updated subgroups in
    // the device-resident mode with the downscale fused (host_io mirrors the
    // working copy into the host image instead)
    ring_phase = ring_cfg().on && fuse && !S.host_io && S.host_updates != 0 && wait_fn && wait_value_ok;
    if (ring_phase && (!ring_mem || ring_threads < dos_host_threads())) {
      const RingCfg& rc = ring_cfg();
      if (ring_mem) cudaFreeHost(ring_mem);
      ring_threads = dos_host_threads();
      const size_t bytes = (size_t)ring_threads * rc.slots * rc.chunk * 2;
      DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&ring_mem), bytes, cudaHostAllocMapped));
      void* dptr = nullptr;
      DOS_CU(cudaHostGetDevicePointer(&dptr, ring_mem, 0));
      ring_mem_dev = static_cast<uint16_t*>(dptr);
      ring_last.assign((size_t)ring_threads * rc.slots, -1);
    }
    // the grad ring: in-phase flush of 16-bit grads, the host lane's slices
    // laid out for the team it will run on
    gring_phase = gring_cfg().on && S.flush_grads && !S.host_io && S.host_updates != 0 && wait_fn && write_fn &&
                  wait_value_ok && !ring_phase;
    if (gring_phase) {
      const GRingCfg& gc = gring_cfg();
      const int team = dos_host_threads();
      gring_k = host_threads > 0 ? std::min(host_threads, team) : team;
      const size_t bytes = (size_t)gc.slots * gring_k * gc.chunk * 2;
      if (bytes > gring_bytes) {
        if (gring_mem) cudaFreeHost(gring_mem);
        gring_mem = nullptr;
        DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&gring_mem), bytes, cudaHostAllocDefault));
        gring_bytes = bytes;
      }
      if (!gring_flags) {
        DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&gring_flags), 2 * 64 * 4, cudaHostAllocMapped));
        memset(gring_flags, 0, 2 * 64 * 4);
        void* dptr = nullptr;
        DOS_CU(cudaHostGetDevicePointer(&dptr, gring_flags, 0));
        gring_flags_dev = (CUdeviceptr)dptr;
        gring_seq = 0;
      }
      gring_counts.assign(gc.slots, 0);
    }
    if (ring_phase && !sh_ctl) {
      DOS_CU(cudaHostAlloc(reinterpret_cast<void**>(&sh_ctl), sizeof(dos_shuttle_ctl), cudaHostAllocMapped));
      memset(sh_ctl, 0, sizeof(dos_shuttle_ctl));
      void* dptr = nullptr;
      DOS_CU(cudaHostGetDevicePointer(&dptr, sh_ctl, 0));
      sh_ctl_dev = static_cast<dos_shuttle_ctl*>(dptr);
    }
    if (ring_phase) {
      // launched before anything of this phase is queued anywhere: no stream's
      // pending wait can sit in front of it
      __atomic_store_n(&sh_ctl->stop, 0u, __ATOMIC_RELEASE);
      sh_phase_first = sh_next.load();
      const int ctas = ring_cfg().ctas;
      const int rc = dos_shuttle_launch(sh_ctl_dev, reinterpret_cast<uint32_t*>(ring_flags_dev), sh_phase_first, ctas,
                                        wst);
      if (rc != DOS_OK) return rc;
      sh_running = true;
      dos_reserve_sms(ctas);
    }
    max_actions = cap;
    count = 0;
    is_host.assign(cap, 0);
    host_done.assign(cap, 0);
    host_s.assign(cap, 0);
    host_e.assign(cap, 0);
    sg_slot.assign(ns, -1);
    sg_mask.assign(ns, 0);
    next_slot = 0;
    slot_release[0] = slot_release[1] = -1;
    slot_owner[0] = slot_owner[1] = -1;
    err = DOS_OK;
    errmsg.clear();
    host_err = DOS_OK;
    host_errmsg.clear();
    DOS_CU(cudaEventRecord(ev0, st[0]));
    DOS_CU(cudaStreamWaitEvent(st[1], ev0, 0));
    DOS_CU(cudaStreamWaitEvent(st[2], ev0, 0));
    DOS_CU(cudaStreamWaitEvent(gst, ev0, 0));
    DOS_CU(cudaStreamWaitEvent(ost, ev0, 0));
    DOS_CU(cudaStreamWaitEvent(pst, ev0, 0));
    flush_q.clear();
    if (S.host_io) {
      // static residents' grads go H2D first thing, on the side stream, so
      // their updates (STATIC_LAST: at the end of the phase) never wait on them
      while ((int)ev_sg.size() < ns) {
        cudaEvent_t e;
        DOS_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_sg.push_back(e);
      }
      static_q.clear();
      for (int i = 0; i < ns && S.host_io_ahead <= 0; ++i)
        if (static_off[i] >= 0) {
          DOS_CU(copy_grads_h2d(sg_start[i], sg_size[i], gst));
          DOS_CU(cudaEventRecord(ev_sg[i], gst));
        }
    }
    DOS_CU(cudaEventSynchronize(ev0));
    host_t0 = now_ns();
    active = true;
    return DOS_OK;
  }

  int finish(int64_t* start_ns, int64_t* end_ns, int32_t n) {
    if (!active) return dos_set_error(DOS_ESTATE, "dos_exec_finish without an active phase");
    {
      std::unique_lock<std::mutex> lk(mu);
      done_cv.wait(lk, [&] { return inflight == 0; });
    }
    sh_stop();  // the host lane posted everything: the shuttle drains and exits
    active = false;
    cudaError_t ce = cudaSuccess;
    for (int i = 0; i < 7; ++i) {
      cudaError_t e = cudaStreamSynchronize(i < 3 ? st[i] : i == 3 ? gst : i == 4 ? ost : i == 5 ? pst : wst);
      if (e != cudaSuccess && ce == cudaSuccess) ce = e;
    }
    dos_reserve_sms(0);
    if (ce != cudaSuccess) return dos_set_error(DOS_ECUDA, "update phase failed on the device: %s", cudaGetErrorString(ce));
    if (host_err != DOS_OK) return dos_set_error(host_err, "host lane: %s", host_errmsg.c_str());
    if (err != DOS_OK) return dos_set_error(err, "%s", errmsg.c_str());
    for (int i = 0; i < 2; ++i)
      if (slot_release[i] == -2)
        return dos_set_error(DOS_ESTATE, "staging store not drained: subgroup %d", slot_owner[i]);
    const int32_t k = std::min(n, count);
    for (int32_t i = 0; i < k; ++i) {
      if (is_host[i]) {
        start_ns[i] = host_s[i];
        end_ns[i] = host_e[i];
      } else {
        float ms_s = 0.f, ms_e = 0.f;
        DOS_CU(cudaEventElapsedTime(&ms_s, ev0, ev_s[i]));
        DOS_CU(cudaEventElapsedTime(&ms_e, ev0, ev_e[i]));
        start_ns[i] = (int64_t)((double)ms_s * 1e6);
        end_ns[i] = (int64_t)((double)ms_e * 1e6);
      }
    }
    return DOS_OK;
  }

  int create(const dos_exec_config* c) {
    dev = c->device;
    nslots = c->num_slots;
    slot_elems = c->slot_elems;
    fuse = c->fuse_downscale != 0;
    host_threads = c->host_threads;
    if (nslots < 1 || nslots > 2) return dos_set_error(DOS_EINVAL, "num_slots must be 1 or 2");
    if (slot_elems < 0) return dos_set_error(DOS_EINVAL, "slot_elems must be >= 0");
    DOS_CU(cudaSetDevice(dev));
    for (int i = 0; i < 3; ++i) DOS_CU(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    DOS_CU(cudaStreamCreateWithFlags(&gst, cudaStreamNonBlocking));
    DOS_CU(cudaStreamCreateWithFlags(&ost, cudaStreamNonBlocking));
    DOS_CU(cudaStreamCreateWithFlags(&pst, cudaStreamNonBlocking));
    DOS_CU(cudaStreamCreateWithFlags(&wst, cudaStreamNonBlocking));
    DOS_CU(cudaEventCreate(&ev0));
    if (slot_elems > 0) DOS_CU(cudaMalloc(reinterpret_cast<void**>(&slot_mem), (size_t)nslots * 3 * slot_elems * 4));
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      wait_fn = reinterpret_cast<pfn_wait_value32>(fn);
    else
      cudaGetLastError();
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      write_fn = reinterpret_cast<pfn_write_value32>(fn);
    else
      cudaGetLastError();
    worker = std::thread([this] { worker_loop(); });
    return DOS_OK;
  }

  void destroy() {
    if (sh_ctl) sh_stop();
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (worker.joinable()) worker.join();
    cudaSetDevice(dev);
    for (int i = 0; i < 3; ++i)
      if (st[i]) {
        cudaStreamSynchronize(st[i]);
        cudaStreamDestroy(st[i]);
      }
    for (cudaStream_t side : {gst, ost, pst, wst})
      if (side) {
        cudaStreamSynchronize(side);
        cudaStreamDestroy(side);
      }
    for (int d = 0; d < 2; ++d) {
      for (int h = 0; h < 7; ++h) {
        if (hst[d][h]) {
          cudaStreamSynchronize(hst[d][h]);
          cudaStreamDestroy(hst[d][h]);
        }
        if (sev_join[d][h]) cudaEventDestroy(sev_join[d][h]);
      }
      if (sev_fork[d]) cudaEventDestroy(sev_fork[d]);
    }
    for (auto e : ev_s) cudaEventDestroy(e);
    for (auto e : ev_e) cudaEventDestroy(e);
    for (auto e : ev_g) cudaEventDestroy(e);
    for (auto e : ev_sg) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (slot_mem) cudaFree(slot_mem);
    if (flags) cudaFreeHost(flags);
    if (ring_flags) cudaFreeHost(ring_flags);
    if (ring_mem) cudaFreeHost(ring_mem);
    if (sh_ctl) cudaFreeHost(sh_ctl);
    if (gring_mem) cudaFreeHost(gring_mem);
    if (gring_flags) cudaFreeHost(gring_flags);
  }
};

}  // namespace

extern "C" int dos_exec_create(const dos_exec_config* cfg, void** out) {
  if (!cfg || !out) return dos_set_error(DOS_EINVAL, "NULL config or out");
  *out = nullptr;
  Engine* e = new Engine();
  const int rc = e->create(cfg);
  if (rc != DOS_OK) {
    std::string msg = dos_last_error();
    e->destroy();
    delete e;
    return dos_set_error(rc, "%s", msg.c_str());
  }
  *out = e;
  return DOS_OK;
}

extern "C" int dos_exec_destroy(void* ex) {
  if (!ex) return DOS_OK;
  Engine* e = static_cast<Engine*>(ex);
  e->destroy();
  delete e;
  return DOS_OK;
}

extern "C" int dos_exec_begin(void* ex, const dos_state_desc* st, const dos_adam_scalars* s, int32_t max_actions) {
  if (!ex) return dos_set_error(DOS_EINVAL, "NULL engine");
  return static_cast<Engine*>(ex)->begin(st, s, max_actions);
}

extern "C" int dos_exec_submit(void* ex, const dos_action_desc* a) {
  if (!ex || !a) return dos_set_error(DOS_EINVAL, "NULL engine or action");
  return static_cast<Engine*>(ex)->submit(a);
}

extern "C" int dos_exec_finish(void* ex, int64_t* start_ns, int64_t* end_ns, int32_t n) {
  if (!ex) return dos_set_error(DOS_EINVAL, "NULL engine");
  if (n > 0 && (!start_ns || !end_ns)) return dos_set_error(DOS_EINVAL, "NULL output arrays");
  return static_cast<Engine*>(ex)->finish(start_ns, end_ns, n);
}

extern "C" int dos_exec_stream_wait(void* ex, int32_t id, void* stream) {
  if (!ex) return dos_set_error(DOS_EINVAL, "NULL engine");
  Engine* e = static_cast<Engine*>(ex);
  if (!e->active) return dos_set_error(DOS_ESTATE, "no active phase");
  if (id < 0 || id >= e->count) return dos_set_error(DOS_EINVAL, "action %d was not submitted", id);
  if (e->is_host[id]) return dos_set_error(DOS_EINVAL, "action %d runs on the host lane (no device event)", id);
  const cudaError_t r = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e->ev_e[id], 0);
  if (r != cudaSuccess) return dos_set_error(DOS_ECUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(r));
  return DOS_OK;
}

extern "C" int dos_exec_slot_ptr(void* ex, int32_t slot, int32_t piece, float** out) {
  if (!ex || !out) return dos_set_error(DOS_EINVAL, "NULL engine or out");
  Engine* e = static_cast<Engine*>(ex);
  if (slot < 0 || slot >= e->nslots || piece < 0 || piece > 2) return dos_set_error(DOS_EINVAL, "bad slot/piece");
  *out = e->slot_ptr(slot, piece);
  return DOS_OK;
}
