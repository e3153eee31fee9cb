// Host runtime of the B200 sampling sweep and the C ABI declared in include/mpsg.h.
//
// One handle holds the compressed MPS resident on each listed device (data-parallel replicas,
// the reference's run_data_parallel, parallel.cpp:240-330, without the per-site broadcast since
// every replica keeps the whole chain in HBM).  mpsg_sample splits [first, first+count) into
// contiguous per-device ranges, each driven by its own host thread and CUDA stream; per device the
// range is cut into passes of `cap` samples and each pass runs the site loop of
// detail::sample_micro_serial (sampler.cpp:129-162) as two kernels per site:
//   K1 site_gemm (tcgen05 contraction + fused weight/max epilogue), K2 select (draw, CDF, gather,
//   renormalise, split).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/mpsg.h"
#include "internal.hpp"
#include "sweep.cuh"

namespace mpsg {

// ---------------------------------------------------------------------------------------------
// errors (errors.hpp:8-27 mapped to codes)
// ---------------------------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

#define CUDA_OK(expr)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw Error(MPSG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
  } while (0)

void check_launch(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(MPSG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static void config_check(bool ok, const std::string& msg) {
  if (!ok) throw Error(MPSG_ERR_CONFIG, msg);
}

// ---------------------------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda link dependency)
// ---------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw Error(MPSG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// fp16 matrix [rows][cols] (cols contiguous), box box_k cols x box_rows rows; 64-wide boxes use
// the 128 B swizzle, 32-wide ones the 64 B swizzle.
static CUtensorMap make_tma_2d(const void* base, uint64_t cols, uint64_t rows,
                               uint32_t box_rows = kBM, uint32_t box_k = kBK) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_k, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_k == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MPSG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// temp [rows][d][chirp] float2 as a 3-D tensor {chirp, d, rows} of 8-byte elements: box 32 columns x
// 1 outcome x 8 samples (the K1 epilogue's TMA tensor stores, 256 B contiguous per sample).
static CUtensorMap make_tma_temp(const void* base, uint64_t chirp, uint64_t d, uint64_t rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {chirp, d, rows};
  cuuint64_t strides[2] = {chirp * 8, d * chirp * 8};
  cuuint32_t box[3] = {32, 1, 8};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MPSG_ERR_CUDA, "cuTensorMapEncodeTiled (temp) failed");
  return m;
}

// Shard-major env [shards][planes * cap rows][kshard]: box 32 k x box_rows rows x 1 shard.
static CUtensorMap make_tma_env(const void* base, uint64_t kshard, uint64_t rows, uint64_t shards,
                                uint32_t box_rows = kBM, uint32_t box_k = kBK) {
  CUtensorMap m;
  cuuint64_t dims[3] = {kshard, rows, shards};
  cuuint64_t strides[2] = {kshard * 2, rows * kshard * 2};
  cuuint32_t box[3] = {box_k, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_k == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MPSG_ERR_CUDA, "cuTensorMapEncodeTiled (3d) failed");
  return m;
}

// Column shard [begin, end) of part `i` of `extent` over `parts`: the reference's balanced_partition
// (collective.cpp:80-92) rounded to whole K blocks of `granule` columns -- every shard but the last
// has round_up(ceil(extent / parts), granule) columns.  A shard of site i's columns is the env K
// shard of site i + 1; with block-aligned shards the K position of every row l is l itself, so the
// contraction accumulates exactly the K blocks of the unsharded sweep in the same order (zero
// blocks appended at most) and a tensor-parallel handle samples bit-identically to an unsharded one.
static void part_range(int extent, int parts, int i, int& b, int& e, int granule) {
  if (parts <= 1) {
    b = 0;
    e = extent;
    return;
  }
  const int a = round_up((extent + parts - 1) / parts, granule);
  b = std::min(i * a, extent);
  e = std::min(b + a, extent);
}

// ---------------------------------------------------------------------------------------------
// collectives for tensor parallelism: NCCL (dlopen'd) or an in-process group of handles
// ---------------------------------------------------------------------------------------------
struct Comm {
  virtual ~Comm() = default;
  // In place: this rank's chunk sits at buf + rank * chunk; afterwards every slot is filled.
  // lane: the pipeline lane issuing the call; every lane has its own ordered channel (its own NCCL
  // communicator) so the two lanes' collectives never interleave on one communicator.
  virtual void allgather(void* buf, size_t chunk, cudaStream_t s, int lane) = 0;
  // Strided all-gather: rank q's data are the byte runs [q * stride + off, + len) of buf, for every
  // (off, len) in runs; afterwards every rank holds every rank's runs (the rest of buf untouched).
  virtual void allgather_runs(void* buf, size_t stride, const std::vector<std::pair<size_t, size_t>>& runs,
                              cudaStream_t s, int lane) = 0;
};

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.commSplit = reinterpret_cast<decltype(api.commSplit)>(dlsym(h, "ncclCommSplit"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.commCount = reinterpret_cast<decltype(api.commCount)>(dlsym(h, "ncclCommCount"));
  });
  if (!api.allGather || !api.commInitRank || !api.getUniqueId || !api.broadcast || !api.groupStart ||
      !api.groupEnd)
    throw Error(MPSG_ERR_CUDA, "NCCL (libnccl.so.2) not available");
  return api;
}

#define NCCL_OK(expr)                                                                 \
  do {                                                                                \
    ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                            \
      throw Error(MPSG_ERR_CUDA, std::string(#expr) + ": " + nccl().getErrorString(r_)); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm[2] = {nullptr, nullptr};  // lane 0, lane 1 (split from lane 0 on first use)
  int rank = 0, nranks = 1;
  NcclComm(const ncclUniqueId& id, int n, int r) : rank(r), nranks(n) {
    NCCL_OK(nccl().commInitRank(&comm[0], nranks, id, r));
  }
  ncclComm_t lane_comm(int lane) {
    if (lane == 1 && !comm[1]) {  // collective: every rank reaches it at the same point of the sweep
      if (!nccl().commSplit) throw Error(MPSG_ERR_CUDA, "ncclCommSplit unavailable (needs NCCL >= 2.18)");
      NCCL_OK(nccl().commSplit(comm[0], 0, rank, &comm[1], nullptr));
    }
    return comm[lane];
  }
  void allgather_runs(void* buf, size_t stride, const std::vector<std::pair<size_t, size_t>>& runs,
                      cudaStream_t s, int lane) override {
    // one broadcast per (root, run), issued as a group: the runs of every root travel concurrently
    ncclComm_t c = lane_comm(lane);
    NCCL_OK(nccl().groupStart());
    for (int q = 0; q < nranks; ++q)
      for (const auto& run : runs) {
        char* p = static_cast<char*>(buf) + q * stride + run.first;
        NCCL_OK(nccl().broadcast(p, p, run.second, ncclUint8, q, c, s));
      }
    NCCL_OK(nccl().groupEnd());
  }
  ~NcclComm() override {
    for (auto c : comm)
      if (c && nccl().commDestroy) nccl().commDestroy(c);
  }
  void allgather(void* buf, size_t chunk, cudaStream_t s, int lane) override {
    ncclComm_t c = lane_comm(lane);
    NCCL_OK(nccl().allGather(static_cast<char*>(buf) + rank * chunk, buf, chunk, ncclUint8, c, s));
  }
};

// Several handles in one process (one per rank, possibly on the same device): the all-gather is
// peer/device copies ordered with events; host threads meet at a barrier twice per call.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<void*> bufs;
  std::vector<int> devices;
  std::vector<cudaEvent_t> ready, done;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
  ~LocalGroup() {
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : done) cudaEventDestroy(e);
  }
};

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  int rank;
  LocalComm(std::shared_ptr<LocalGroup> grp, int r) : g(std::move(grp)), rank(r) {}
  void allgather(void* buf, size_t chunk, cudaStream_t s, int lane) override {
    allgather_runs(buf, chunk, {{0, chunk}}, s, lane);
  }
  void allgather_runs(void* buf, size_t stride, const std::vector<std::pair<size_t, size_t>>& runs,
                      cudaStream_t s, int /*lane*/) override {
    // host barriers serialise the calls of all lanes in issue order, identical on every rank
    LocalGroup& G = *g;
    G.bufs[rank] = buf;
    CUDA_OK(cudaEventRecord(G.ready[rank], s));
    G.barrier();
    for (int q = 0; q < G.n; ++q) {
      if (q == rank) continue;
      CUDA_OK(cudaStreamWaitEvent(s, G.ready[q], 0));
      for (const auto& run : runs)
        CUDA_OK(cudaMemcpyPeerAsync(static_cast<char*>(buf) + q * stride + run.first, G.devices[rank],
                                    static_cast<char*>(G.bufs[q]) + q * stride + run.first, G.devices[q],
                                    run.second, s));
    }
    CUDA_OK(cudaEventRecord(G.done[rank], s));
    G.barrier();
    for (int q = 0; q < G.n; ++q)
      if (q != rank) CUDA_OK(cudaStreamWaitEvent(s, G.done[q], 0));
  }
};

// ---------------------------------------------------------------------------------------------
// power-of-two bond scales gamma_i[r] ~ Lambda_i[r]
// ---------------------------------------------------------------------------------------------
static double pow2_near(double x) {
  int e;
  std::frexp(x, &e);  // x = f 2^e, f in [0.5,1)
  e = std::max(-60, std::min(60, e - 1));
  return std::ldexp(1.0, e);
}
static std::vector<double> bond_scales(const double* lambda, size_t n) {
  std::vector<double> g(n, 1.0);
  double last = 1.0;
  for (size_t r = 0; r < n; ++r) {
    if (lambda[r] > 0.0 && std::isfinite(lambda[r])) last = pow2_near(lambda[r]);
    g[r] = last;
  }
  return g;
}

// ---------------------------------------------------------------------------------------------
// storage-streamed Gamma (mpsg_create_from_file_streamed): the reference's SiteStream
// (mps_io.cpp:294-350) as a pass-by-pass supply.  A reader thread preads the MPSB site payloads in
// chain order (sites 0..M-1, repeated every pass) into a ring of pinned staging buffers and verifies
// their FNV-1a checksums (mps_io.cpp:120-146); the copy stream uploads the raw Gamma scalars and the
// compression kernels pack them into the device slot the sweep consumes next.
// ---------------------------------------------------------------------------------------------
struct FileMeta {
  std::string path;
  std::vector<uint64_t> off, bytes, check;  // per site: payload offset, payload bytes, checksum
  std::vector<int> prec;                    // per site: storage precision (MPSG_F64 / F32 / F16)
  std::vector<uint64_t> gbytes;             // per site: Gamma scalar bytes (payload minus Lambda)
};

static uint64_t fnv1a64(const uint8_t* p, size_t n) {  // mps_io.cpp:18-25
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

// pread of one site payload + checksum verification; throws Error(MPSG_ERR_IO)
static void read_payload(int fd, const FileMeta& fm, uint64_t i, uint8_t* dst) {
  size_t got = 0;
  const size_t want = fm.bytes[i];
  while (got < want) {
    const ssize_t r = ::pread(fd, dst + got, want - got, static_cast<off_t>(fm.off[i] + got));
    if (r <= 0) throw Error(MPSG_ERR_IO, "mps file truncated at site " + std::to_string(i) + ": " + fm.path);
    got += static_cast<size_t>(r);
  }
  if (fnv1a64(dst, want) != fm.check[i])
    throw Error(MPSG_ERR_IO, "mps file corrupt: checksum mismatch at site " + std::to_string(i));
}

// R staging buffers and R reader threads: load q (site q % M) goes to buffer q % R, and the threads
// work on the R loads after the consumer's position concurrently -- the per-payload FNV-1a is a
// byte-serial chain (~1 GB/s per thread), so one reader would cap the stream at ~1 GB/s.
struct FileReader {
  const FileMeta* fm = nullptr;
  int device = 0;
  int fd = -1;
  int R = 2;
  std::vector<uint8_t*> stage;       // pinned, max payload bytes each
  std::vector<cudaEvent_t> copied;   // the upload from stage[b] is done (recorded by the consumer)
  std::vector<long long> holds;      // load sequence number held by stage[b] (-1: none)
  std::vector<long long> inflight;   // load sequence number being read into stage[b] (-1: none)
  long long next = 0;                // the next sequence number the consumer takes
  bool stop = false;
  std::string err;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::thread> th;

  FileReader(const FileMeta& meta, int dev) : fm(&meta), device(dev) {
    fd = ::open(meta.path.c_str(), O_RDONLY);
    if (fd < 0) throw Error(MPSG_ERR_IO, "cannot open: " + meta.path);
    (void)::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
    uint64_t mx = 1;
    for (uint64_t b : meta.bytes) mx = std::max(mx, b);
    // up to 8 buffers / threads within 8 GiB of pinned staging, at least 2 (double buffering)
    R = static_cast<int>(std::max<uint64_t>(2, std::min<uint64_t>(8, (8ull << 30) / mx)));
    stage.assign(R, nullptr);
    copied.assign(R, nullptr);
    holds.assign(R, -1);
    inflight.assign(R, -1);
    for (int b = 0; b < R; ++b) {
      CUDA_OK(cudaMallocHost(&stage[b], mx));
      CUDA_OK(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
    }
    for (int t = 0; t < R; ++t) th.emplace_back([this] { run(); });
  }
  ~FileReader() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th)
      if (t.joinable()) t.join();
    for (int b = 0; b < R; ++b) {
      if (stage[b]) cudaFreeHost(stage[b]);
      if (copied[b]) cudaEventDestroy(copied[b]);
    }
    if (fd >= 0) ::close(fd);
  }
  void run() {
    cudaSetDevice(device);
    const long long m = static_cast<long long>(fm->off.size());
    for (;;) {
      long long q = 0;
      {
        std::unique_lock<std::mutex> lk(mu);
        auto pick = [&] {
          for (q = next; q < next + R; ++q)
            if (holds[q % R] != q && inflight[q % R] != q) return true;
          return false;
        };
        cv.wait(lk, [&] { return stop || (err.empty() && pick()); });
        if (stop) return;
        holds[q % R] = -1;
        inflight[q % R] = q;
      }
      const int b = static_cast<int>(q % R);
      std::string e;
      try {
        CUDA_OK(cudaEventSynchronize(copied[b]));  // the previous upload from this buffer is done
        read_payload(fd, *fm, static_cast<uint64_t>(q % m), stage[b]);
      } catch (const std::exception& x) {
        e = x.what();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        inflight[b] = -1;
        if (e.empty())
          holds[b] = q;
        else
          err = e;
      }
      cv.notify_all();
    }
  }
  // Blocks until the payload of load q (site q % M) is staged; q must be the next in sequence.
  const uint8_t* take(long long q) {
    std::unique_lock<std::mutex> lk(mu);
    if (q != next) throw Error(MPSG_ERR_INTERNAL, "file site stream out of sequence");
    cv.wait(lk, [&] { return holds[q % R] == q || !err.empty(); });
    if (holds[q % R] != q) throw Error(MPSG_ERR_IO, err);
    return stage[q % R];
  }
  // The upload from load q's staging buffer was enqueued on `s`.
  void taken(long long q, cudaStream_t s) {
    CUDA_OK(cudaEventRecord(copied[q % R], s));
    {
      std::lock_guard<std::mutex> lk(mu);
      next = q + 1;
    }
    cv.notify_all();
  }
};

// ---------------------------------------------------------------------------------------------
// state
// ---------------------------------------------------------------------------------------------
struct SiteDev {
  int chil = 0, chir = 0, kp = 0, chirp = 0, np = 0, nt = 0;
  int b0 = 0, width = 0;     // this rank's column shard [b0, b0 + width) of chiR
  int kshard = 0;            // env K extent per shard (kp = shards * kshard)
  __half* g = nullptr;       // [gplanes][np][kp]
  float2* cinfo = nullptr;   // [np]
  double* cs = nullptr;      // [chir * d]
  double* inv_gamma = nullptr;  // [width] 1 / gamma_i[r] of the local columns (decay trace)
  CUtensorMap tma_g{}, tma_g64{};
  // generated supply: base isometry id and the per-site factors of the generator
  int base_id = -1;
  float* lam_prev_f = nullptr;  // [chil] fp32 Lambda_{i-1}
  float* inv_lam_f = nullptr;   // [chir] fp32 1 / Lambda_i
  double *gl_d = nullptr, *gr_d = nullptr, *wl_d = nullptr;  // bond scales, weight factors
  int* lpos_d = nullptr;        // [chil] K position of row l
  // host-streamed mode: the compressed site lives in pinned host memory
  __half* g_host = nullptr;
  float2* cinfo_host = nullptr;
  std::vector<CUtensorMap> tma_slot, tma_slot64;  // G maps per device slot
};

// One pipeline lane: a sample range of the pass with its own buffers and stream.  With two lanes
// the contraction kernels of the lanes are ordered alternately (A_i, B_i, A_i+1, ...) while each
// lane's select kernel runs underneath the other lane's contraction.
struct Lane {
  cudaStream_t stream = nullptr;  // lane 0 uses DevCtx::stream
  int cap = 0;                    // rows, multiple of 256
  __half* env = nullptr;          // [shards][2 * env_comp][cap][kshard_max]
  float2* temp = nullptr;         // [cap][d][chirp_max]
  float2* pstat = nullptr;        // [cap][nt_max]
  float2* part = nullptr;         // [tp][cap][d] exchanged (weight, max) partials (TP only)
  uint8_t* alive = nullptr;       // [cap]
  uint8_t* rows = nullptr;        // [cap][M]
  uint8_t* forced = nullptr;      // [cap][M] (lazy)
  double* marg = nullptr;         // [cap][M][d] (lazy)
  double* logscale = nullptr;     // [cap] (lazy, decay trace)
  double2* mu = nullptr;          // [cap][M] displacement amplitudes of the pass (lazy)
  uint8_t* host_rows = nullptr;   // pinned [cap][M]
  std::vector<CUtensorMap> tma_env;    // per site: the shard-major env map over this lane's env
  std::vector<CUtensorMap> tma_env64;  // same with a 64-row box (3M kernel: env is the B operand)
  std::vector<CUtensorMap> tma_temp;   // per site: temp as {chirp, d, cap} (K1's TMA tensor stores)
  // slice-recompute path (3M, tp = 1): rows bucketed by outcome each site
  __half* env_perm = nullptr;     // the environment rows in bucket order (slice GEMM B operand)
  int* perm = nullptr;            // [cap] row -> sample of the pass
  int* perm2 = nullptr;
  uint8_t* rowk = nullptr;        // [cap] drawn outcome per row (d = dead from the next site)
  float* scale = nullptr;         // [cap] renormalisation per row
  float* scale2 = nullptr;        // [cap] the same in bucket order
  uint8_t* alive2 = nullptr;
  int* bcount = nullptr;          // [2 (d + 1)] bucket counts, fill cursors
  std::vector<CUtensorMap> tma_envp64;  // per site: B maps over env_perm
  cudaEvent_t k1done = nullptr, done = nullptr;
  cudaEvent_t seldone = nullptr;  // this lane's selection of the current site (host-streamed slots)
  std::vector<cudaEvent_t> gev;   // per-site contraction start/stop, slice GEMM start/stop (4 M)
};

struct DevCtx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::vector<SiteDev> sites;
  int cap = 0;               // pass capacity (rows over all lanes)
  std::vector<Lane> lanes;
  double* scratch = nullptr; // compress: gl, gr, wl
  void* src = nullptr;       // compress staging (device)
  size_t src_bytes = 0;
  int* err = nullptr;
  unsigned long long* colmax = nullptr;  // [chirp_max * d] compression scratch (kept zeroed)
  // generated supply (mpsg_generated_*): base isometries and the per-site phase buffer
  std::vector<float2*> bases;
  std::vector<long long> base_rows, base_cols;
  float2* phase = nullptr;
  std::vector<long long> slot_sig;  // extents of each slot's last fill (its padding is zero)
  // storage-streamed supply (mpsg_create_from_file_streamed): staging reader + raw device buffers
  std::unique_ptr<FileReader> reader;
  std::vector<void*> slot_raw;
  std::vector<cudaEvent_t> raw_ready;  // the raw upload into slot_raw[q] is done (copy stream)
  // host-streamed Gamma: ring of device slots filled by a copy stream (sequence q -> slot q % R)
  int slots = 0;
  std::vector<__half*> slot_g;
  std::vector<float2*> slot_cinfo;
  std::vector<cudaEvent_t> loaded, freed;
  cudaStream_t copy_stream = nullptr;
  uint64_t issued = 0, consumed = 0;  // rolling site-load sequence (sites 0..M-1, repeated)
  uint64_t h2d_bytes = 0;
  std::vector<cudaEvent_t> ev;   // per-site boundaries on lane 0 (M + 1)
  cudaEvent_t pass_end = nullptr;
  double* trace = nullptr;       // [M] sum |env_ref| per site (decay trace, lazy)
  unsigned long long* live = nullptr;  // [M] live samples measured per site (RunStats counters)
  unsigned long long* near = nullptr;  // [M] draws within kBoundaryEps of a CDF boundary per site
};

}  // namespace mpsg

struct mpsg_handle_s {
  uint64_t M = 0, d = 0;
  std::vector<uint64_t> bonds;
  mpsg_policy policy{};
  mpsg_options opts{};
  bool split = true;
  std::vector<std::vector<double>> gl, gr;  // per site: left / right bond scales
  std::vector<std::vector<double>> lambda;  // Lambda_i as given (MPSB save, reporting)
  std::vector<mpsg::DevCtx> devs;
  std::vector<char> site_set;
  bool finished = false;
  int tp = 1, tp_rank = 0;                 // tensor-parallel group (column-sharded Gamma)
  bool pair = true;                        // K1 variant: CTA-pair UMMA (M=256) vs A-multicast pairs
  bool m3 = false;                         // 3M contraction (Gamma planes Gr, Gi, Gs; env re, im, s)
  int gplanes = 2, env_comp = 2;
  // planes kept per site in pinned host memory when Gamma is host-streamed: the 3M sum planes
  // (Gs = Gr + Gi, exact by construction) are re-formed on the device after the copy, so the host
  // link carries 4 B per complex entry for 3M as for 4M (PRECISE: 8 of the 12 B)
  int hplanes = 2;
  bool precise = false;                    // Gamma hi + lo planes (MPSG_MODE_PRECISE)
  bool slice_rc = false;                   // slice-recompute path available (3M, tp = 1, d <= 32)
  int grid = 0;                            // kGrid*: MPSG_MODE_GRID (the TF32 / F16 policies' grids)
  bool precise_auto = false;               // MPSG_MODE_AUTO at F64 / F32: PRECISE if its state fits
  bool generated = false;                  // Gamma regenerated on the device every pass (synthetic chains)
  uint64_t gen_seed = 0;
  bool file = false;                       // Gamma streamed from an MPSB file every pass
  // 3M with only [Gr, Gi] resident in HBM (the 3-plane state does not fit, the 2-plane one does):
  // every site is copied device-to-device into the slot ring and its Gs plane re-formed there
  // (the host-streamed machinery with device memory as the store)
  bool dev_store = false;
  mpsg::FileMeta fmeta;
  std::unique_ptr<mpsg::Comm> comm;
  std::mutex mu;
};

namespace mpsg {

// N-tile pairs per raster group: the group's Gamma tiles (<= 2 x 16 x 1 MiB at chi = 2048) stay in
// L2 across the M sweep while the env tiles are re-read once per group.
constexpr int kGroupPairs = 16;

// K block of the contraction: env shards and Gamma column shards are aligned to it (part_range)
static int kgran(const mpsg_handle_s& h) { return h.m3 ? kBK3 : kBK; }
static int kshard_of(const mpsg_handle_s& h, uint64_t bond) {
  return round_up((static_cast<int>(bond) + h.tp - 1) / h.tp, kgran(h));
}
static int kshard_max_of(const mpsg_handle_s& h) {
  int k = kBK;
  for (uint64_t i = 0; i < h.M; ++i) k = std::max(k, kshard_of(h, h.bonds[i]));
  return k;
}
static int chirp_of(const mpsg_handle_s& h, uint64_t bond) {
  return round_up((static_cast<int>(bond) + h.tp - 1) / h.tp, kBN);
}
static int chirp_max_of(const mpsg_handle_s& h) {
  int c = kBN;
  for (uint64_t i = 1; i <= h.M; ++i) c = std::max(c, chirp_of(h, h.bonds[i]));
  return c;
}

// 3M unless asked otherwise, the A-multicast 4M variant was selected, or the 3-plane state does not
// fit: next to the pass buffers in device memory (resident) or in host memory (host-streamed; the
// stream then carries 1.5x the bytes of 4M, measured at 96% of the resident c3 rate).
static void choose_scheme(mpsg_handle_s& h) {
  bool m3 = h.opts.scheme != MPSG_SCHEME_4M;
  if (h.grid) {  // per-component grids: Gr + Gi is not on the grid, so no 3M sum plane
    config_check(h.opts.scheme != MPSG_SCHEME_3M, "MPSG_MODE_GRID runs the 4M scheme (Gr + Gi is off the grid)");
    m3 = false;
  } else if (h.opts.scheme == MPSG_SCHEME_AUTO && (h.generated || h.file)) {
    m3 = h.pair;  // regenerated / streamed into device slots: no state to fit
  } else if (h.opts.scheme == MPSG_SCHEME_AUTO) {
    if (!h.pair) m3 = false;
    double state3 = 0.0, max_site3 = 0.0;
    for (uint64_t i = 0; i < h.M; ++i) {
      const double kp = static_cast<double>(h.tp) * kshard_of(h, h.bonds[i]);
      const double np = round_up(static_cast<int>(h.d) * chirp_of(h, h.bonds[i + 1]), 2 * kBN);
      state3 += 3.0 * 2.0 * np * kp;
      max_site3 = std::max(max_site3, 3.0 * 2.0 * np * kp);
    }
    if (h.opts.host_stream_slots != 0) {
      const double host = static_cast<double>(sysconf(_SC_PHYS_PAGES)) * sysconf(_SC_PAGE_SIZE);
      if (state3 * (2.0 / 3.0) * h.devs.size() > 0.8 * host) m3 = false;  // host keeps Gr, Gi only
    } else {
      bool compact = m3;
      for (auto& dc : h.devs) {
        size_t free_b = 0, total_b = 0;
        CUDA_OK(cudaSetDevice(dc.device));
        CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
        if (state3 + 10.0e9 > static_cast<double>(free_b)) m3 = false;  // pass buffers + headroom
        // [Gr, Gi] resident + a 3-slot ring of 3-plane sites (MPSG_COMPACT_3M=0 disables)
        if (state3 * (2.0 / 3.0) + 3.0 * max_site3 + 12.0e9 > static_cast<double>(free_b)) compact = false;
      }
      // MPSG_COMPACT_3M: 0 = never, 1 = when only the 2-plane state fits (default), 2 = always (tests)
      static const int env_compact = [] {
        const char* v = std::getenv("MPSG_COMPACT_3M");
        return v == nullptr ? 1 : std::atoi(v);
      }();
      if (h.pair && (!m3 || env_compact == 2) && compact && env_compact != 0 && !h.precise_auto && h.tp == 1 &&
          h.opts.mode != MPSG_MODE_PRECISE) {
        m3 = true;
        h.dev_store = true;
        h.opts.host_stream_slots = 3;
      }
    }
  }
  if (h.precise_auto) {  // MPSG_MODE_AUTO at compute F64 / F32: PRECISE when its 6 planes fit
    double state6 = 0.0;
    for (uint64_t i = 0; i < h.M; ++i)
      state6 += 6.0 * 2.0 * round_up(static_cast<int>(h.d) * chirp_of(h, h.bonds[i + 1]), 2 * kBN) *
                static_cast<double>(h.tp) * round_up((static_cast<int>(h.bonds[i]) + h.tp - 1) / h.tp, kBK3);
    bool fits = h.pair && h.opts.scheme != MPSG_SCHEME_4M;
    if (h.file || h.generated) {
      // streamed from storage / regenerated: only the slot ring is resident, whatever the chain's size
    } else if (h.opts.host_stream_slots != 0) {
      const double host = static_cast<double>(sysconf(_SC_PHYS_PAGES)) * sysconf(_SC_PAGE_SIZE);
      fits = fits && state6 * (4.0 / 6.0) * h.devs.size() <= 0.6 * host;
    } else {
      for (auto& dc : h.devs) {
        size_t free_b = 0, total_b = 0;
        CUDA_OK(cudaSetDevice(dc.device));
        CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
        fits = fits && state6 + 10.0e9 <= static_cast<double>(free_b);
      }
    }
    h.precise = fits;
  }
  if (h.precise) {
    config_check(h.opts.scheme != MPSG_SCHEME_4M, "MPSG_MODE_PRECISE needs the 3M scheme");
    m3 = true;
    double state6 = 0.0;  // 6 Gamma planes: fail early with the sizes
    for (uint64_t i = 0; i < h.M; ++i)
      state6 += 6.0 * 2.0 * round_up(static_cast<int>(h.d) * chirp_of(h, h.bonds[i + 1]), 2 * kBN) *
                static_cast<double>(h.tp) * round_up((static_cast<int>(h.bonds[i]) + h.tp - 1) / h.tp, kBK3);
    if (h.file || h.generated) {
      // only the slot ring is resident
    } else if (h.opts.host_stream_slots != 0) {
      const double host = static_cast<double>(sysconf(_SC_PHYS_PAGES)) * sysconf(_SC_PAGE_SIZE);
      config_check(state6 * (4.0 / 6.0) * h.devs.size() <= 0.85 * host,
                   "MPSG_MODE_PRECISE: the hi + lo Gamma planes need " + std::to_string(state6 * 4.0 / 6.0 / 1e9) +
                       " GB of pinned host memory per device");
    } else {
      for (auto& dc : h.devs) {
        size_t free_b = 0, total_b = 0;
        CUDA_OK(cudaSetDevice(dc.device));
        CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
        config_check(state6 + 4.0e9 <= static_cast<double>(free_b),
                     "MPSG_MODE_PRECISE: the hi + lo Gamma planes need " + std::to_string(state6 / 1e9) +
                         " GB of device memory; use host_stream_slots or tensor parallelism");
      }
    }
  }
  h.m3 = m3;
  h.gplanes = h.precise ? 6 : (m3 ? 3 : 2);
  h.hplanes = m3 ? h.gplanes * 2 / 3 : h.gplanes;
  h.env_comp = m3 ? 3 : 2;
}

static void validate_shape(uint64_t m, uint64_t d, const uint64_t* bonds) {
  // MpsState::validate (mps.cpp:12-20) + GPU-path limits
  config_check(m > 0, "mps has no sites");
  config_check(d >= 1, "mps physical dimension must be >= 1");
  config_check(d <= 254, "phys_dim must fit the u8 outcome encoding (<= 254)");
  config_check(bonds != nullptr, "bond_dims is null");
  config_check(bonds[0] == 1 && bonds[m] == 1, "boundary bonds must be 1");
  for (uint64_t i = 0; i <= m; ++i) {
    config_check(bonds[i] >= 1, "bond dimensions must be >= 1");
    config_check(bonds[i] <= (1u << 20), "bond dimension too large for the device format");
  }
}

static void validate_policy(const mpsg_policy& p) {
  config_check(p.compute >= MPSG_F64 && p.compute <= MPSG_F16, "unknown compute precision");
  config_check(p.storage >= MPSG_F64 && p.storage <= MPSG_F16, "unknown storage precision");
  // PrecisionPolicy::validate (precision.cpp:98-102)
  config_check(p.storage != MPSG_TF32, "storage precision must be one of f64/f32/f16");
  config_check(p.scaling >= MPSG_SCALE_NONE && p.scaling <= MPSG_SCALE_PER_SAMPLE_MAX,
               "unknown scaling mode");
}

static void validate_lambda(const double* lam, size_t n) {
  // mps.cpp:30-36
  for (size_t j = 0; j < n; ++j) {
    if (lam[j] < 0.0) throw Error(MPSG_ERR_NUMERIC, "lambda entries must be nonnegative");
    if (j > 0 && lam[j] > lam[j - 1])
      throw Error(MPSG_ERR_NUMERIC, "lambda vectors must be nonincreasing");
  }
}

static void alloc_device(mpsg_handle_s& h, DevCtx& dc) {
  CUDA_OK(cudaSetDevice(dc.device));
  int major = 0;
  CUDA_OK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dc.device));
  if (major != 10) throw Error(MPSG_ERR_CUDA, "device is not sm_100 (B200)");
  CUDA_OK(cudaDeviceGetAttribute(&dc.num_sms, cudaDevAttrMultiProcessorCount, dc.device));
  // Stream priorities: the lanes' streams (contraction, selection) run at the device's greatest
  // priority and the copy stream (slot copies, Gs re-formation, side-stream compression) at its
  // least, so the block scheduler places a persistent contraction's CTAs before further supply blocks
  int prio_least = 0, prio_greatest = 0;
  CUDA_OK(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
  CUDA_OK(cudaStreamCreateWithPriority(&dc.stream, cudaStreamNonBlocking, prio_greatest));
  const int kmax = h.tp * kshard_max_of(h), chirpm = chirp_max_of(h);
  const size_t nt_max = h.d * (chirpm / kBN) + 1;  // + the pair-padding tile
  const size_t row_bytes = 4ull * h.env_comp * kmax + 8ull * h.d * chirpm + 8ull * nt_max + 1 + h.M +
                           (h.tp > 1 ? 8ull * h.tp * h.d : 0);
  uint64_t want = h.opts.pass_samples;
  if (want == 0) {
    const double budget = 6.0e9;  // bytes of per-pass working set
    want = std::min<uint64_t>(65536, static_cast<uint64_t>(budget / row_bytes));
  }
  // Two lanes overlap the select kernel with the other lane's contraction (a selection block fits
  // next to the 128-register 3M contraction on an SM).  Measured (profiles/r1_lanes_ab/, one box,
  // alternating runs): c3 +1.9%, chi = 512 / 256 neutral, so two lanes for chains with chi >= 1024.
  // Tensor parallelism always uses two lanes: one lane's partial / environment all-gathers and
  // selection run underneath the other lane's contraction, so the GEMM and the collectives overlap.
  uint64_t chi_max = 1;
  for (uint64_t i = 0; i <= h.M; ++i) chi_max = std::max(chi_max, h.bonds[i]);
  int nlanes = (h.tp > 1 || (h.m3 && chi_max >= 1024)) ? 2 : 1;
  if (const char* v = std::getenv("MPSG_LANES")) nlanes = std::max(1, std::min(2, std::atoi(v)));
  // host-streamed Gamma: both lanes read each slot; the slice-recompute path keeps one lane
  if (h.opts.host_stream_slots != 0 && h.opts.slice == MPSG_SLICE_RECOMPUTE) nlanes = 1;
  const int lane_cap = std::max(2 * kBM, round_up(static_cast<int>((std::min<uint64_t>(want, 1u << 22) +
                                                                     nlanes - 1) / nlanes), 2 * kBM));
  dc.cap = nlanes * lane_cap;
  dc.sites.resize(h.M);
  dc.lanes.resize(nlanes);
  for (int L = 0; L < nlanes; ++L) {
    Lane& ln = dc.lanes[L];
    ln.cap = lane_cap;
    if (L == 0)
      ln.stream = dc.stream;
    else
      CUDA_OK(cudaStreamCreateWithPriority(&ln.stream, cudaStreamNonBlocking, prio_greatest));
    CUDA_OK(cudaMalloc(&ln.env, 2ull * h.env_comp * ln.cap * kmax * sizeof(__half)));
    CUDA_OK(cudaMalloc(&ln.temp, 1ull * ln.cap * h.d * chirpm * sizeof(float2)));
    CUDA_OK(cudaMalloc(&ln.pstat, 1ull * ln.cap * nt_max * sizeof(float2)));

    CUDA_OK(cudaMalloc(&ln.alive, ln.cap));
    CUDA_OK(cudaMalloc(&ln.rows, 1ull * ln.cap * h.M));
    CUDA_OK(cudaMallocHost(&ln.host_rows, 1ull * ln.cap * h.M));
    CUDA_OK(cudaEventCreateWithFlags(&ln.k1done, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ln.done, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&ln.seldone, cudaEventDisableTiming));
    ln.tma_env.resize(h.M);
    ln.tma_env64.resize(h.M);
    ln.tma_temp.resize(h.M);
    if (h.slice_rc) {
      CUDA_OK(cudaMalloc(&ln.env_perm, 2ull * h.env_comp * ln.cap * kmax * sizeof(__half)));
      CUDA_OK(cudaMalloc(&ln.perm, ln.cap * sizeof(int)));
      CUDA_OK(cudaMalloc(&ln.perm2, ln.cap * sizeof(int)));
      CUDA_OK(cudaMalloc(&ln.rowk, ln.cap));
      CUDA_OK(cudaMalloc(&ln.scale, ln.cap * sizeof(float)));
      CUDA_OK(cudaMalloc(&ln.scale2, ln.cap * sizeof(float)));
      CUDA_OK(cudaMalloc(&ln.alive2, ln.cap));
      CUDA_OK(cudaMalloc(&ln.bcount, 2 * (h.d + 1) * sizeof(int)));
      ln.tma_envp64.resize(h.M);
    }
  }
  CUDA_OK(cudaMalloc(&dc.err, sizeof(int)));
  CUDA_OK(cudaMemset(dc.err, 0, sizeof(int)));
  CUDA_OK(cudaMalloc(&dc.colmax, sizeof(unsigned long long) * chirpm * h.d));
  CUDA_OK(cudaMemset(dc.colmax, 0, sizeof(unsigned long long) * chirpm * h.d));
  if (h.generated) {
    uint64_t cols = 1;
    for (uint64_t i = 1; i <= h.M; ++i) cols = std::max(cols, h.bonds[i] * h.d);
    CUDA_OK(cudaMalloc(&dc.phase, sizeof(float2) * cols));
  }
  CUDA_OK(cudaMalloc(&dc.scratch, sizeof(double) * (kmax + 2ull * h.tp * chirpm) + sizeof(int) * kmax));
  if (h.opts.host_stream_slots > 0) {
    config_check(h.opts.host_stream_slots >= 2, "host_stream_slots must be 0 or >= 2");
    dc.slots = h.opts.host_stream_slots;
    size_t gmax = 0, nmax = 0;
    for (uint64_t i = 0; i < h.M; ++i) {
      const size_t kp = static_cast<size_t>(h.tp) * kshard_of(h, h.bonds[i]);
      const size_t np = round_up(static_cast<int>(h.d) * chirp_of(h, h.bonds[i + 1]), 2 * kBN);
      gmax = std::max(gmax, static_cast<size_t>(h.gplanes) * np * kp);
      nmax = std::max(nmax, np);
    }
    CUDA_OK(cudaStreamCreateWithPriority(&dc.copy_stream, cudaStreamNonBlocking, prio_least));
    dc.slot_g.resize(dc.slots);
    dc.slot_cinfo.resize(dc.slots);
    dc.loaded.resize(dc.slots);
    dc.freed.resize(dc.slots);
    for (int q = 0; q < dc.slots; ++q) {
      CUDA_OK(cudaMalloc(&dc.slot_g[q], gmax * sizeof(__half)));
      CUDA_OK(cudaMalloc(&dc.slot_cinfo[q], nmax * sizeof(float2)));
      CUDA_OK(cudaEventCreateWithFlags(&dc.loaded[q], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&dc.freed[q], cudaEventDisableTiming));
    }
    dc.slot_sig.assign(dc.slots, -1);
    if (h.file) {  // raw Gamma scalars of a site as stored in the file, one buffer per slot
      uint64_t rmax = 1;
      for (uint64_t g : h.fmeta.gbytes) rmax = std::max(rmax, g);
      dc.slot_raw.assign(dc.slots, nullptr);
      dc.raw_ready.assign(dc.slots, nullptr);
      for (int q = 0; q < dc.slots; ++q) {
        CUDA_OK(cudaMalloc(&dc.slot_raw[q], rmax));
        CUDA_OK(cudaEventCreateWithFlags(&dc.raw_ready[q], cudaEventDisableTiming));
      }
      dc.reader = std::make_unique<FileReader>(h.fmeta, dc.device);
    }
  }
}

static void free_device(DevCtx& dc) {
  cudaSetDevice(dc.device);
  if (dc.stream) cudaStreamSynchronize(dc.stream);
  if (dc.copy_stream) cudaStreamSynchronize(dc.copy_stream);
  dc.reader.reset();  // joins the reader thread
  for (auto p : dc.slot_raw) cudaFree(p);
  dc.slot_raw.clear();
  for (auto e : dc.raw_ready) cudaEventDestroy(e);
  dc.raw_ready.clear();
  for (auto& s : dc.sites) {
    if (!dc.slots) {
      cudaFree(s.g);
      cudaFree(s.cinfo);
    }
    cudaFree(s.cs);
  }
  for (auto& ln : dc.lanes) {
    if (ln.stream && ln.stream != dc.stream) {
      cudaStreamSynchronize(ln.stream);
      cudaStreamDestroy(ln.stream);
    }
    cudaFree(ln.env);
    cudaFree(ln.temp);
    cudaFree(ln.pstat);
    cudaFree(ln.part);
    cudaFree(ln.alive);
    cudaFree(ln.rows);
    cudaFree(ln.forced);
    cudaFree(ln.marg);
    cudaFree(ln.logscale);
    cudaFree(ln.mu);
    cudaFree(ln.env_perm);
    cudaFree(ln.perm);
    cudaFree(ln.perm2);
    cudaFree(ln.rowk);
    cudaFree(ln.scale);
    cudaFree(ln.scale2);
    cudaFree(ln.alive2);
    cudaFree(ln.bcount);
    if (ln.host_rows) cudaFreeHost(ln.host_rows);
    if (ln.k1done) cudaEventDestroy(ln.k1done);
    if (ln.done) cudaEventDestroy(ln.done);
    if (ln.seldone) cudaEventDestroy(ln.seldone);
    for (auto e : ln.gev) cudaEventDestroy(e);
  }
  cudaFree(dc.scratch);
  cudaFree(dc.src);
  cudaFree(dc.err);
  cudaFree(dc.colmax);
  cudaFree(dc.phase);
  for (auto p : dc.bases) cudaFree(p);
  for (auto& s : dc.sites) {
    cudaFree(s.lam_prev_f);
    cudaFree(s.inv_lam_f);
    cudaFree(s.gl_d);
    cudaFree(s.gr_d);
    cudaFree(s.wl_d);
    cudaFree(s.lpos_d);
  }
  cudaFree(dc.trace);
  cudaFree(dc.live);
  cudaFree(dc.near);
  for (auto& s : dc.sites) cudaFree(s.inv_gamma);
  for (auto e : dc.ev) cudaEventDestroy(e);
  if (dc.pass_end) cudaEventDestroy(dc.pass_end);
  if (dc.copy_stream) cudaStreamSynchronize(dc.copy_stream);
  for (auto& s : dc.sites) {
    for (void* p : {static_cast<void*>(s.g_host), static_cast<void*>(s.cinfo_host)}) {
      if (!p) continue;
      cudaPointerAttributes at = {};  // the store: pinned host memory, or device memory (compact 3M)
      if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice)
        cudaFree(p);
      else
        cudaFreeHost(p);
    }
    if (dc.slots) s.g = nullptr, s.cinfo = nullptr;  // slot buffers, freed below
  }
  for (auto p : dc.slot_g) cudaFree(p);
  for (auto p : dc.slot_cinfo) cudaFree(p);
  for (auto e : dc.loaded) cudaEventDestroy(e);
  for (auto e : dc.freed) cudaEventDestroy(e);
  if (dc.copy_stream) cudaStreamDestroy(dc.copy_stream);
  if (dc.stream) cudaStreamDestroy(dc.stream);
}

// Site geometry of this rank's column shard of site i (padded extents, shard range) and its
// per-site device arrays that do not depend on the Gamma values.
static void site_geometry(mpsg_handle_s& h, DevCtx& dc, uint64_t i) {
  SiteDev& s = dc.sites[i];
  s.chil = static_cast<int>(h.bonds[i]);
  s.chir = static_cast<int>(h.bonds[i + 1]);
  part_range(s.chir, h.tp, h.tp_rank, s.b0, s.width, kgran(h));
  s.width -= s.b0;
  s.kshard = kshard_of(h, h.bonds[i]);
  s.kp = h.tp * s.kshard;
  s.chirp = chirp_of(h, h.bonds[i + 1]);
  s.np = round_up(static_cast<int>(h.d) * s.chirp, 2 * kBN);  // whole N-tile pairs (CTA pairs)
  s.nt = s.np / kBN;
  if (!s.cs) CUDA_OK(cudaMalloc(&s.cs, std::max<size_t>(1, 1ull * s.width * h.d) * sizeof(double)));
  if (!s.inv_gamma) CUDA_OK(cudaMalloc(&s.inv_gamma, std::max<size_t>(1, s.width) * sizeof(double)));
  std::vector<double> ig(std::max(1, s.width));
  for (int r = 0; r < s.width; ++r) ig[r] = 1.0 / h.gr[i][s.b0 + r];
  CUDA_OK(cudaMemcpy(s.inv_gamma, ig.data(), sizeof(double) * ig.size(), cudaMemcpyHostToDevice));
}

// K position of row l: the previous site's column shards, each padded to kshard
static std::vector<int> row_positions(const mpsg_handle_s& h, const SiteDev& s) {
  std::vector<int> lpos(s.chil);
  for (int q = 0; q < h.tp; ++q) {
    int b, e;
    part_range(s.chil, h.tp, q, b, e, kgran(h));
    for (int l = b; l < e; ++l) lpos[l] = q * s.kshard + (l - b);
  }
  return lpos;
}

// weight factors wl_r = (Lambda_i[r] / gamma_i[r])^2 of the Born weights
static std::vector<double> weight_factors(const mpsg_handle_s& h, uint64_t i, const double* lambda) {
  std::vector<double> wl(h.bonds[i + 1]);
  for (size_t r = 0; r < wl.size(); ++r) {
    const double q = lambda[r] / h.gr[i][r];
    wl[r] = q * q;
  }
  return wl;
}

// TMA maps of site i: the environment of every lane and the Gamma planes (resident or per slot).
static void site_maps(mpsg_handle_s& h, DevCtx& dc, uint64_t i) {
  SiteDev& s = dc.sites[i];
  for (auto& ln : dc.lanes) {
    const uint64_t env_rows = 2ull * h.env_comp * ln.cap;
    ln.tma_env[i] = make_tma_env(ln.env, s.kshard, env_rows, h.tp);
    if (h.m3) ln.tma_env64[i] = make_tma_env(ln.env, s.kshard, env_rows, h.tp, kBM / 2, kBK3);
    if (h.m3) ln.tma_temp[i] = make_tma_temp(ln.temp, s.chirp, h.d, ln.cap);
    if (ln.env_perm) ln.tma_envp64[i] = make_tma_env(ln.env_perm, s.kshard, env_rows, h.tp, kBM / 2, kBK3);
  }
  if (dc.slots) {
    s.tma_slot.resize(dc.slots);
    s.tma_slot64.resize(dc.slots);
    for (int q = 0; q < dc.slots; ++q) {
      s.tma_slot[q] = make_tma_2d(dc.slot_g[q], s.kp, static_cast<uint64_t>(h.gplanes) * s.np, kBM,
                                  h.m3 ? kBK3 : kBK);
      s.tma_slot64[q] = make_tma_2d(dc.slot_g[q], s.kp, static_cast<uint64_t>(h.gplanes) * s.np, kBN / 2);
    }
  } else {
    s.tma_g = make_tma_2d(s.g, s.kp, static_cast<uint64_t>(h.gplanes) * s.np, kBM, h.m3 ? kBK3 : kBK);
    s.tma_g64 = make_tma_2d(s.g, s.kp, static_cast<uint64_t>(h.gplanes) * s.np, kBN / 2);
  }
}

static void check_err_flag(DevCtx& dc, cudaStream_t stream, const std::string& where) {
  int err = 0;
  CUDA_OK(cudaMemcpyAsync(&err, dc.err, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CUDA_OK(cudaStreamSynchronize(stream));
  if (err != 0) {
    cudaMemset(dc.err, 0, sizeof(int));
    throw Error(MPSG_ERR_NUMERIC, "contract_site: non-finite input (" + where +
                                      ") or dynamic range beyond the compressed format");
  }
}

// Compress this rank's column shard of site i on device dc from `src` (device pointer).
static void compress_site(mpsg_handle_s& h, DevCtx& dc, uint64_t i, const void* src_dev,
                          bool f64, const double* lambda) {
  SiteDev& s = dc.sites[i];
  site_geometry(h, dc, i);
  if (dc.slots) {  // compress into slot 0, then keep the result in pinned host memory
    CUDA_OK(cudaStreamSynchronize(dc.copy_stream));
    s.g = dc.slot_g[0];
    s.cinfo = dc.slot_cinfo[0];
  } else if (!s.g) {
    CUDA_OK(cudaMalloc(&s.g, static_cast<size_t>(h.gplanes) * s.np * s.kp * sizeof(__half)));
    CUDA_OK(cudaMalloc(&s.cinfo, 1ull * s.np * sizeof(float2)));
  }
  const std::vector<double> wl = weight_factors(h, i, lambda);
  const std::vector<int> lpos = row_positions(h, s);
  double* d_gl = dc.scratch;
  double* d_gr = d_gl + s.chil;
  double* d_wl = d_gr + s.chir;
  int* d_lpos = reinterpret_cast<int*>(d_wl + s.chir);
  CUDA_OK(cudaMemcpyAsync(d_gl, h.gl[i].data(), sizeof(double) * s.chil, cudaMemcpyHostToDevice, dc.stream));
  CUDA_OK(cudaMemcpyAsync(d_gr, h.gr[i].data(), sizeof(double) * s.chir, cudaMemcpyHostToDevice, dc.stream));
  CUDA_OK(cudaMemcpyAsync(d_wl, wl.data(), sizeof(double) * s.chir, cudaMemcpyHostToDevice, dc.stream));
  CUDA_OK(cudaMemcpyAsync(d_lpos, lpos.data(), sizeof(int) * s.chil, cudaMemcpyHostToDevice, dc.stream));
  CUDA_OK(cudaMemsetAsync(s.g, 0, static_cast<size_t>(h.gplanes) * s.np * s.kp * sizeof(__half), dc.stream));
  CUDA_OK(cudaMemsetAsync(s.cinfo, 0, 1ull * s.np * sizeof(float2), dc.stream));
  launch_compress_site(src_dev, f64 ? kSrcF64 : kSrcF32, s.chil, s.chir, static_cast<int>(h.d), s.b0, s.width, s.kp,
                       s.chirp, d_lpos, d_gl, d_gr, d_wl, h.gplanes, s.g, s.cinfo, s.cs, dc.colmax, dc.err,
                       dc.stream, h.grid);
  CUDA_OK(cudaGetLastError());
  check_err_flag(dc, dc.stream, "site " + std::to_string(i));
  if (dc.slots) {
    const size_t pe = static_cast<size_t>(s.np) * s.kp;  // elements per plane
    if (!s.g_host) {  // the store: pinned host memory, or device memory for the compact-3M state
      if (h.dev_store) {
        CUDA_OK(cudaMalloc(&s.g_host, h.hplanes * pe * sizeof(__half)));
        CUDA_OK(cudaMalloc(&s.cinfo_host, 1ull * s.np * sizeof(float2)));
      } else {
        CUDA_OK(cudaMallocHost(&s.g_host, h.hplanes * pe * sizeof(__half)));
        CUDA_OK(cudaMallocHost(&s.cinfo_host, 1ull * s.np * sizeof(float2)));
      }
    }
    if (h.hplanes == h.gplanes) {
      CUDA_OK(cudaMemcpyAsync(s.g_host, s.g, h.gplanes * pe * sizeof(__half), cudaMemcpyDefault, dc.stream));
    } else {  // 3M: [Gr, Gi] of each precision half (the Gs planes are re-formed after the slot copy)
      for (int hf = 0; hf < h.gplanes / 3; ++hf)
        CUDA_OK(cudaMemcpyAsync(s.g_host + 2ull * hf * pe, s.g + 3ull * hf * pe, 2 * pe * sizeof(__half),
                                cudaMemcpyDefault, dc.stream));
    }
    CUDA_OK(cudaMemcpyAsync(s.cinfo_host, s.cinfo, 1ull * s.np * sizeof(float2), cudaMemcpyDefault, dc.stream));
    CUDA_OK(cudaStreamSynchronize(dc.stream));
    s.g = nullptr;
    s.cinfo = nullptr;
    dc.issued = dc.consumed = 0;  // slot 0 was overwritten: restart the load sequence
    dc.slot_sig.assign(dc.slots, -1);
  }
  site_maps(h, dc, i);
}

// Generated supply: the generator of site i (base isometry, phases, fp32 Lambda factors) for this
// rank's shard, as the compression kernels read it.
static SynthSite synth_of(const mpsg_handle_s& h, const DevCtx& dc, uint64_t i) {
  const SiteDev& s = dc.sites[i];
  SynthSite g;
  g.base = dc.bases[s.base_id];
  g.ld = dc.base_cols[s.base_id];
  g.cols = static_cast<long long>(s.chir) * static_cast<long long>(h.d);
  g.phase = dc.phase;
  g.lam_prev = s.lam_prev_f;
  g.inv_lam = s.inv_lam_f;
  g.d = static_cast<int>(h.d);
  return g;
}

// Regenerates and compresses site i into device planes g_out / cinfo_out on `stream` (generated
// supply): phases, column maxima and scales, packed fp16 planes -- the same kernels and rounding as
// compressing the materialised site (mpsg_synthetic_site + mpsg_builder_set_site).
static void regenerate_site(const mpsg_handle_s& h, DevCtx& dc, uint64_t i, __half* g_out, float2* cinfo_out,
                            bool clear, cudaStream_t stream) {
  SiteDev& s = dc.sites[i];
  if (clear) {
    CUDA_OK(cudaMemsetAsync(g_out, 0, static_cast<size_t>(h.gplanes) * s.np * s.kp * sizeof(__half), stream));
    CUDA_OK(cudaMemsetAsync(cinfo_out, 0, 1ull * s.np * sizeof(float2), stream));
  }
  launch_synth_phase(h.gen_seed, i, s.chir * static_cast<int>(h.d), dc.phase, stream);
  launch_compress_synth(synth_of(h, dc, i), s.chil, static_cast<int>(h.d), s.b0, s.width, s.kp, s.chirp,
                        s.lpos_d, s.gl_d, s.gr_d, s.wl_d, h.gplanes, g_out, cinfo_out, s.cs, dc.colmax, dc.err,
                        stream);
  check_launch(cudaGetLastError(), "site regeneration");
}

// Host-streamed mode: issue site loads until `upto` loads are in flight or done.
// Stream of the supply's compression kernels (regeneration, file-site packing).  Inline (default):
// the engine's lane-0 stream, between the sites' contractions.  On the side copy stream those kernels
// would interleave with the persistent contraction, whose CTAs own whole SMs with a static unit split:
// CTAs that start late behind a compression block stretch the whole launch (chi = 8192 regenerated:
// +38% per site on the side stream against the kernels' own 1.7 ms, profiles/r2_bigchi/).
static cudaStream_t supply_stream(const DevCtx& dc) {
  static const bool side = [] {
    const char* v = std::getenv("MPSG_SUPPLY_STREAM");
    return v && std::string(v) == "side";
  }();
  return side ? dc.copy_stream : dc.stream;
}

static void issue_loads(mpsg_handle_s& h, DevCtx& dc, uint64_t upto) {
  while (dc.issued < upto) {
    const uint64_t q = dc.issued;
    const int slot = static_cast<int>(q % dc.slots);
    const SiteDev& s = dc.sites[q % h.M];
    CUDA_OK(cudaStreamWaitEvent(dc.copy_stream, dc.freed[slot], 0));  // consume q - slots done
    if (h.file || h.generated) {  // compressed on the device into the slot
      const cudaStream_t ss = supply_stream(dc);
      if (ss != dc.copy_stream) CUDA_OK(cudaStreamWaitEvent(ss, dc.freed[slot], 0));
      // the slot's padding is zero from its last fill when that had the same extents
      const long long sig = (static_cast<long long>(s.np) << 32) ^ (static_cast<long long>(s.kp) << 8) ^
                            (static_cast<long long>(s.chil) * 131 + s.width);
      if (h.file) {  // storage -> pinned staging (reader threads) -> device raw -> compressed slot
        const uint64_t i = q % h.M;
        const uint8_t* raw = dc.reader->take(static_cast<long long>(q));
        CUDA_OK(cudaMemcpyAsync(dc.slot_raw[slot], raw, h.fmeta.gbytes[i], cudaMemcpyHostToDevice, dc.copy_stream));
        dc.reader->taken(static_cast<long long>(q), dc.copy_stream);
        CUDA_OK(cudaEventRecord(dc.raw_ready[slot], dc.copy_stream));
        CUDA_OK(cudaStreamWaitEvent(ss, dc.raw_ready[slot], 0));
        if (dc.slot_sig[slot] != sig) {
          CUDA_OK(cudaMemsetAsync(dc.slot_g[slot], 0, static_cast<size_t>(h.gplanes) * s.np * s.kp * sizeof(__half),
                                  ss));
          CUDA_OK(cudaMemsetAsync(dc.slot_cinfo[slot], 0, 1ull * s.np * sizeof(float2), ss));
        }
        launch_compress_site(dc.slot_raw[slot], h.fmeta.prec[i], s.chil, s.chir, static_cast<int>(h.d), s.b0,
                             s.width, s.kp, s.chirp, s.lpos_d, s.gl_d, s.gr_d, s.wl_d, h.gplanes, dc.slot_g[slot],
                             dc.slot_cinfo[slot], s.cs, dc.colmax, dc.err, ss, h.grid);
        check_launch(cudaGetLastError(), "file site compression");
        dc.h2d_bytes += h.fmeta.gbytes[i];
      } else {  // regenerate + compress on the device: no host traffic
        regenerate_site(h, dc, q % h.M, dc.slot_g[slot], dc.slot_cinfo[slot], dc.slot_sig[slot] != sig, ss);
      }
      dc.slot_sig[slot] = sig;
      CUDA_OK(cudaEventRecord(dc.loaded[slot], ss));
      ++dc.issued;
      continue;
    }
    const size_t pe = static_cast<size_t>(s.np) * s.kp;
    const size_t gb = h.hplanes * pe * sizeof(__half);
    if (h.hplanes == h.gplanes) {
      CUDA_OK(cudaMemcpyAsync(dc.slot_g[slot], s.g_host, gb, cudaMemcpyDefault, dc.copy_stream));
    } else {
      for (int hf = 0; hf < h.gplanes / 3; ++hf) {
        __half* dst = dc.slot_g[slot] + 3ull * hf * pe;
        CUDA_OK(cudaMemcpyAsync(dst, s.g_host + 2ull * hf * pe, 2 * pe * sizeof(__half),
                                cudaMemcpyDefault, dc.copy_stream));
        launch_sum_plane(dst, pe, dc.copy_stream);  // Gs = Gr + Gi (exact fp16 sums)
      }
    }
    CUDA_OK(cudaMemcpyAsync(dc.slot_cinfo[slot], s.cinfo_host, 1ull * s.np * sizeof(float2),
                            cudaMemcpyDefault, dc.copy_stream));
    CUDA_OK(cudaEventRecord(dc.loaded[slot], dc.copy_stream));
    if (!h.dev_store) dc.h2d_bytes += gb + 1ull * s.np * sizeof(float2);
    ++dc.issued;
  }
}

static void ensure_src(DevCtx& dc, size_t bytes) {
  if (dc.src_bytes >= bytes) return;
  cudaFree(dc.src);
  dc.src = nullptr;
  CUDA_OK(cudaMalloc(&dc.src, bytes));
  dc.src_bytes = bytes;
}

static void set_site(mpsg_handle_s& h, uint64_t i, const void* gamma, bool is_device, int dtype,
                     const double* lambda) {
  config_check(!h.finished, "builder already finished");
  config_check(i < h.M, "site index out of range");
  config_check(gamma != nullptr && lambda != nullptr, "null gamma / lambda");
  config_check(dtype == MPSG_F64 || dtype == MPSG_F32, "gamma dtype must be f64 or f32");
  config_check(!h.generated, "a generated handle takes mpsg_generated_set_site");
  // the left bond scales of site i derive from Lambda_{i-1}: sites are set in chain order
  config_check(i == 0 || h.site_set[i - 1], "sites must be set in increasing order");
  // site i's Lambda fixes the left bond scales site i + 1 was compressed with
  config_check(i + 1 == h.M || !h.site_set[i + 1], "site " + std::to_string(i) +
                                                       " cannot be set again after site i + 1 was set");
  const size_t chir = h.bonds[i + 1];
  validate_lambda(lambda, chir);
  // the F16 grid is absolute: Gamma and the environment keep the reference's own values
  h.gr[i] = h.grid == kGridF16 ? std::vector<double>(chir, 1.0) : bond_scales(lambda, chir);
  h.lambda[i].assign(lambda, lambda + chir);
  if (i + 1 < h.M) h.gl[i + 1] = h.gr[i];
  const size_t elems = 2ull * h.bonds[i] * chir * h.d;
  const size_t bytes = elems * (dtype == MPSG_F64 ? 8 : 4);
  for (size_t di = 0; di < h.devs.size(); ++di) {
    DevCtx& dc = h.devs[di];
    CUDA_OK(cudaSetDevice(dc.device));
    const void* src = gamma;
    if (!is_device || di > 0) {
      ensure_src(dc, bytes);
      if (!is_device) {
        CUDA_OK(cudaMemcpyAsync(dc.src, gamma, bytes, cudaMemcpyHostToDevice, dc.stream));
      } else {
        CUDA_OK(cudaMemcpyPeerAsync(dc.src, dc.device, gamma, h.devs[0].device, bytes, dc.stream));
      }
      src = dc.src;
    }
    compress_site(h, dc, i, src, dtype == MPSG_F64, lambda);
  }
  h.site_set[i] = 1;
}

// Generated supply: site i is regenerated from base isometry `base_id` with Lambda_i = lambda on
// every pass; only the generator's per-site factors are stored.
static void set_site_generated(mpsg_handle_s& h, uint64_t i, int base_id, const double* lambda) {
  config_check(h.generated, "not a generated handle (mpsg_generated_begin)");
  config_check(!h.finished, "builder already finished");
  config_check(i < h.M, "site index out of range");
  config_check(lambda != nullptr, "null lambda");
  config_check(i == 0 || h.site_set[i - 1], "sites must be set in increasing order");
  config_check(i + 1 == h.M || !h.site_set[i + 1], "site " + std::to_string(i) +
                                                       " cannot be set again after site i + 1 was set");
  const size_t chil = h.bonds[i], chir = h.bonds[i + 1];
  config_check(base_id >= 0 && base_id < static_cast<int>(h.devs[0].bases.size()), "unknown base isometry id");
  config_check(h.devs[0].base_rows[base_id] >= static_cast<long long>(chil) &&
                   h.devs[0].base_cols[base_id] >= static_cast<long long>(chir * h.d),
               "base isometry smaller than the site (needs bond[i] rows, bond[i+1] * d columns)");
  validate_lambda(lambda, chir);
  h.gr[i] = bond_scales(lambda, chir);
  h.lambda[i].assign(lambda, lambda + chir);
  if (i + 1 < h.M) h.gl[i + 1] = h.gr[i];
  std::vector<float> lp(chil, 1.0f), il(chir);
  if (i > 0)
    for (size_t l = 0; l < chil; ++l) lp[l] = static_cast<float>(h.lambda[i - 1][l]);
  for (size_t r = 0; r < chir; ++r) il[r] = 1.0f / static_cast<float>(lambda[r]);
  for (auto& dc : h.devs) {
    CUDA_OK(cudaSetDevice(dc.device));
    site_geometry(h, dc, i);
    SiteDev& sd = dc.sites[i];
    sd.base_id = base_id;
    const std::vector<double> wl = weight_factors(h, i, lambda);
    const std::vector<int> lpos = row_positions(h, sd);
    auto up = [](auto*& dst, const auto& v) {
      using T = std::remove_reference_t<decltype(v[0])>;
      if (!dst) CUDA_OK(cudaMalloc(&dst, sizeof(T) * v.size()));
      CUDA_OK(cudaMemcpy(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    };
    up(sd.lam_prev_f, lp);
    up(sd.inv_lam_f, il);
    up(sd.gl_d, h.gl[i]);
    up(sd.gr_d, h.gr[i]);
    up(sd.wl_d, wl);
    up(sd.lpos_d, lpos);
    site_maps(h, dc, i);
  }
  h.site_set[i] = 1;
}

// Storage-streamed supply: site i's bond scales, weight factors and K positions (from Lambda_i, read
// with the header); its Gamma is read from the file and compressed on every pass.
static void set_site_file(mpsg_handle_s& h, uint64_t i, const double* lambda) {
  config_check(h.file, "not a file-streamed handle");
  config_check(i < h.M && (i == 0 || h.site_set[i - 1]), "sites must be set in increasing order");
  const size_t chir = h.bonds[i + 1];
  validate_lambda(lambda, chir);
  h.gr[i] = h.grid == kGridF16 ? std::vector<double>(chir, 1.0) : bond_scales(lambda, chir);
  h.lambda[i].assign(lambda, lambda + chir);
  if (i + 1 < h.M) h.gl[i + 1] = h.gr[i];
  for (auto& dc : h.devs) {
    CUDA_OK(cudaSetDevice(dc.device));
    site_geometry(h, dc, i);
    SiteDev& sd = dc.sites[i];
    const std::vector<double> wl = weight_factors(h, i, lambda);
    const std::vector<int> lpos = row_positions(h, sd);
    auto up = [](auto*& dst, const auto& v) {
      using T = std::remove_reference_t<decltype(v[0])>;
      if (!dst) CUDA_OK(cudaMalloc(&dst, sizeof(T) * v.size()));
      CUDA_OK(cudaMemcpy(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    };
    up(sd.gl_d, h.gl[i]);
    up(sd.gr_d, h.gr[i]);
    up(sd.wl_d, wl);
    up(sd.lpos_d, lpos);
    site_maps(h, dc, i);
  }
  h.site_set[i] = 1;
}

// ---------------------------------------------------------------------------------------------
// the sweep
// ---------------------------------------------------------------------------------------------
struct PassOut {
  uint64_t macs = 0, wmacs = 0, issued = 0, launches = 0, dmacs = 0, pops = 0, near = 0;
  double gemm_s = 0.0, device_s = 0.0;
};

// Where the renormalisation max of the 3M path comes from: the K1 epilogue (tensor parallelism, which
// exchanges it with the weights, and long-K sites, where the epilogue has slack: +1.5% at c3) or the
// select kernel's pass over the chosen slice (short-K sites, where the epilogue is on the critical
// path: +10% at chi = 512).
// The tensor-parallel data plane (partials exchange, environment all-gather) runs for a TP group of
// p2 > 1 ranks, and for a connected one-rank group (the same collectives through NCCL on one GPU).
static bool xchg(const mpsg_handle_s& h) { return h.tp > 1 || h.comm != nullptr; }
static bool epilogue_max(const mpsg_handle_s& h, const SiteDev& s) { return xchg(h) || s.kp >= 1024; }


// K1 for `rows` samples of lane `ln` at site i.  tma_g128 / tma_g64: Gamma maps with 128 / 64-row
// boxes (the 3M kernel loads Gamma as its A operand; the 4M pair kernel as its half-B operand).
// slice: 0 = K1 (temp + weights), 1 = weights only (slice-recompute path), 2 = the slice GEMM
static void launch_contraction(const mpsg_handle_s& h, const DevCtx& dc, const SiteDev& s, const Lane& ln,
                               uint64_t i, int rows, const CUtensorMap* tma_g128,
                               const CUtensorMap& tma_g64, const float2* cinfo, cudaStream_t stream,
                               int slice = 0, int kp_next = 0, bool pdl = false) {
  if (h.m3) {
    Gemm3MArgs ga = {};
    ga.pdl = pdl ? 1 : 0;
    ga.g_tiles = s.np / (2 * kBN);
    ga.s_tiles = rows / kBM;
    ga.k_blocks = s.kp / kBK3;
    ga.kshard_blocks = s.kshard / kBK3;
    ga.env_cap = ln.cap;
    ga.np = s.np;
    ga.chirp = s.chirp;
    ga.d = static_cast<int>(h.d);
    ga.nt = s.nt;
    static const int env_group = [] {
      const char* v = std::getenv("MPSG_3M_GROUP");
      return v ? std::max(1, std::atoi(v)) : 0;
    }();
    // Gamma tile pairs per raster group: as many as fit ~25 MB of Gamma planes, at least 8 (c3:
    // 8 pairs = 25 MB -- larger groups measured more DRAM traffic and less speed, profiles/
    // r1_l2_experiments/; c2 and c5 chi = 1024: the whole site, +2.5%, profiles/r1_group_ab/)
    const double pair_bytes = 2.0 * kBM * s.kp * sizeof(__half) * h.gplanes;
    const int auto_group = std::max(8, static_cast<int>(26214400.0 / pair_bytes));
    static const int env_flags = [] {
      const char* v = std::getenv("MPSG_3M_FLAGS");
      return v ? std::atoi(v) : 0;
    }();
    ga.group = std::min(ga.g_tiles, env_group > 0 ? env_group : auto_group);
    ga.flags = env_flags;
    // L2 reuse across raster groups (snake) and, for the second lane, across the lanes' launches
    static const int env_raster = [] {
      const char* v = std::getenv("MPSG_3M_RASTER");
      return v ? std::atoi(v) : 3;
    }();
    const bool lane1 = &ln != &dc.lanes[0];
    ga.raster = (env_raster & 1) | ((env_raster & 2) && lane1 && ga.g_tiles % ga.group == 0 ? 2 : 0);
    ga.cinfo = cinfo;
    ga.temp = slice == 0 ? ln.temp : nullptr;
    ga.pstat = slice == 2 ? nullptr : ln.pstat;
    if (slice == 2) {
      ga.bcount = ln.bcount;
      ga.scale = ln.scale2;
      ga.env_next = ln.env;
      ga.kp_next = kp_next;
    }
    const int ctas = 2 * ga.g_tiles * ga.s_tiles;
    static const int env_epi = [] {
      const char* v = std::getenv("MPSG_3M_EPI");
      return v ? std::atoi(v) : 8;
    }();
    static const bool env_quad = [] {
      const char* v = std::getenv("MPSG_3M_QUAD");
      return v && std::atoi(v) != 0;
    }();
    // temp through TMA tensor stores (MPSG_3M_TMA_STORE=1: A/B switch)
    static const bool env_tma = [] {
      const char* v = std::getenv("MPSG_3M_TMA_STORE");
      return v && std::atoi(v) != 0;
    }();
    const bool tma_store = env_tma && slice == 0 && !h.precise;
    launch_site_gemm_3m(h.split, slice == 1 || epilogue_max(h, s), env_epi, env_quad && slice == 0, h.precise,
                        slice == 2 ? ln.tma_envp64[i] : ln.tma_env64[i], *tma_g128, ga, std::min(ctas, dc.num_sms),
                        stream, slice == 2, tma_store ? &ln.tma_temp[i] : nullptr);
    return;
  }
  const int mrow = h.pair ? 2 * kBM : kBM;
  SiteGemmArgs ga;
  ga.m_tiles = rows / mrow;
  ga.n_tiles = s.nt;
  ga.k_blocks = s.kp / kBK;
  ga.kshard_blocks = s.kshard / kBK;
  ga.plane_rows_a = ln.cap;
  ga.np = s.np;
  ga.chirp = s.chirp;
  ga.d = static_cast<int>(h.d);
  ga.group_n = h.pair ? std::min(s.nt, 2 * kGroupPairs) : std::min(s.nt / 2, kGroupPairs);
  ga.cinfo = cinfo;
  ga.temp = ln.temp;
  ga.pstat = ln.pstat;
  const int ctas = h.pair ? 2 * ga.m_tiles * ga.n_tiles : ga.m_tiles * ga.n_tiles;
  if (h.pair)
    launch_site_gemm_pair(h.split, ln.tma_env[i], tma_g64, ga, std::min(ctas, dc.num_sms), stream);
  else
    launch_site_gemm(h.split, ln.tma_env[i], *tma_g128, ga, std::min(ctas, dc.num_sms), stream);
}

// Enqueues one pass of `count` (<= dc.cap) samples starting at global index `first`, split over
// the lanes.  Lane L covers [first + off[L], first + off[L] + cnt[L]).
static void run_pass(mpsg_handle_s& h, DevCtx& dc, uint64_t seed, uint64_t first, int count,
                     bool forced, bool marg, bool displaced, PassOut& po, int timing, int off[2],
                     int cnt[2]) {
  const int nl = static_cast<int>(dc.lanes.size());
  const int mrow = (h.pair && !h.m3) ? 2 * kBM : kBM;
  off[0] = 0;
  cnt[0] = count;
  cnt[1] = 0;
  if (nl == 2 && count > 2 * kBM) {  // halves rounded to whole M tiles
    cnt[0] = std::min(dc.lanes[0].cap, round_up((count + 1) / 2, 2 * kBM));
    cnt[1] = count - cnt[0];
  }
  off[1] = cnt[0];
  const int active = cnt[1] > 0 ? 2 : 1;
  // slice recompute for plain sampling passes (teacher forcing, marginals, displacement and the decay
  // trace read temp): rows are then permuted by outcome every such site, perm maps them to samples
  const bool rc_pass = h.slice_rc && !forced && !marg && !displaced && !dc.trace;
  // Programmatic dependent launch between the contraction and the selection of consecutive sites
  // (one lane, HBM-resident Gamma, no exchange / displacement / slice recompute): each
  // kernel's prologue overlaps its predecessor's tail.  Opt-in (MPSG_PDL=1): measured neutral at
  // chi = 256 / 512 (profiles/r2_select_rows/), where the per-site launches are shortest.
  static const bool env_pdl = [] {
    const char* v = std::getenv("MPSG_PDL");
    return v != nullptr && std::atoi(v) != 0;
  }();
  const bool pdl = env_pdl && h.m3 && nl == 1 && !dc.slots && !xchg(h) && !displaced && !rc_pass;
  int rows[2];
  for (int L = 0; L < active; ++L) {
    Lane& ln = dc.lanes[L];
    rows[L] = round_up(cnt[L], mrow);
    if (L > 0 && timing) CUDA_OK(cudaStreamWaitEvent(ln.stream, dc.ev[0], 0));  // after the pass-start stamp
    launch_init_env(ln.env, h.env_comp, ln.cap, dc.sites[0].kshard, h.tp, rows[L], cnt[L], ln.alive,
                    ln.stream, dc.trace ? ln.logscale : nullptr, rc_pass ? ln.perm : nullptr);
    po.launches += 1;
  }
  if (dc.slots) issue_loads(h, dc, dc.consumed + dc.slots);
  for (uint64_t i = 0; i < h.M; ++i) {
    const SiteDev& s = dc.sites[i];
    const CUtensorMap* tma_g128 = &s.tma_g;
    const CUtensorMap* tma_g64 = &s.tma_g64;
    const float2* cinfo = s.cinfo;
    int slot = -1;
    if (dc.slots) {  // single lane in host-streamed mode
      if (dc.consumed % h.M != i) throw Error(MPSG_ERR_INTERNAL, "site stream out of sequence");
      slot = static_cast<int>(dc.consumed % dc.slots);
      CUDA_OK(cudaStreamWaitEvent(dc.stream, dc.loaded[slot], 0));
      tma_g128 = &s.tma_slot[slot];
      tma_g64 = &s.tma_slot64[slot];
      cinfo = dc.slot_cinfo[slot];
    }
    for (int L = 0; L < active; ++L) {
      Lane& ln = dc.lanes[L];
      const uint64_t lfirst = first + off[L];
      static const bool lane_sync = [] {  // MPSG_LANE_SYNC=0: A/B switch (no cross-lane ordering)
        const char* v = std::getenv("MPSG_LANE_SYNC");
        return v == nullptr || std::atoi(v) != 0;
      }();
      if (active == 2 && (lane_sync || dc.slots)) {  // contraction kernels alternate A_i, B_i, A_i+1, ...
        if (L == 1)
          CUDA_OK(cudaStreamWaitEvent(ln.stream, dc.lanes[0].k1done, 0));
        else if (i > 0)
          CUDA_OK(cudaStreamWaitEvent(ln.stream, dc.lanes[1].k1done, 0));
      }
      const bool has_next = i + 1 < h.M;
      const bool rc = rc_pass && h.opts.slice == MPSG_SLICE_RECOMPUTE;
      if (timing >= 2) CUDA_OK(cudaEventRecord(ln.gev[4 * i], ln.stream));
      launch_contraction(h, dc, s, ln, i, rows[L], tma_g128, *tma_g64, cinfo, ln.stream, rc ? 1 : 0, 0, pdl);
      if (timing >= 2) CUDA_OK(cudaEventRecord(ln.gev[4 * i + 1], ln.stream));
      // Displacement fused into the selection (one read of temp) unless the weights must be exchanged
      // first (tensor parallelism) or the decay trace reads the transformed slice.
      static const bool no_fuse = std::getenv("MPSG_DISPLACE_SEPARATE") != nullptr;
      const bool fuse_displace = displaced && !xchg(h) && !dc.trace && !no_fuse && !h.grid;
      if (displaced && !fuse_displace) {  // the SiteTransform hook position (sampler.cpp:143)
        DisplaceArgs da;
        da.d = static_cast<int>(h.d);
        da.chirp = s.chirp;
        da.chir_loc = s.width;
        da.nt = s.nt;
        da.tpk = s.chirp / kBN;
        da.rows = rows[L];
        da.count = cnt[L];
        da.site = static_cast<int>(i);
        da.num_sites = static_cast<int>(h.M);
        da.mu = ln.mu;
        da.alive = ln.alive;
        da.cinfo = cinfo;
        da.temp = ln.temp;
        da.pstat = ln.pstat;
        launch_displace(da, ln.stream);
        po.launches += 1;
      }
      if (active == 2) CUDA_OK(cudaEventRecord(ln.k1done, ln.stream));
      // Host-streamed Gamma: the slot (planes and cinfo) is read by the contraction(s), the fused
      // displacement selection and the slice GEMM of every lane; the last lane hands it back to the
      // copy stream once all of them are done (lane 1's contraction already follows lane 0's).
      auto release_slot = [&] {
        if (!dc.slots || L != active - 1) return;
        if (active == 2) CUDA_OK(cudaStreamWaitEvent(ln.stream, dc.lanes[0].seldone, 0));
        CUDA_OK(cudaEventRecord(dc.freed[slot], ln.stream));
        ++dc.consumed;
        issue_loads(h, dc, dc.consumed + dc.slots);
      };

      SelectArgs sa;
      sa.pdl = pdl ? 1 : 0;
      sa.site = static_cast<int>(i);
      sa.num_sites = static_cast<int>(h.M);
      sa.d = static_cast<int>(h.d);
      sa.chir_loc = s.width;
      sa.chirp = s.chirp;
      if (!xchg(h)) {  // partials straight from the tiles: (tile t of outcome k) at pstat[n][k*tpk+t]
        sa.parts = s.chirp / kBN;
        sa.part_base = ln.pstat;
        sa.part_stride = 1;
        sa.row_stride = s.nt;
        sa.k_stride = s.chirp / kBN;
      } else {  // per-rank (weight, max) per outcome, exchanged, summed in rank order on every rank
        launch_reduce_tiles(ln.pstat, s.nt, s.chirp / kBN, sa.d, rows[L],
                            ln.part + 1ull * h.tp_rank * ln.cap * h.d, ln.stream);
        h.comm->allgather(ln.part, 1ull * ln.cap * h.d * sizeof(float2), ln.stream, L);
        sa.parts = h.tp;
        sa.part_base = ln.part;
        sa.part_stride = 1ll * ln.cap * static_cast<long long>(h.d);
        sa.row_stride = static_cast<long long>(h.d);
        sa.k_stride = 1;
        po.launches += 1;
      }
      sa.rows = rows[L];
      sa.count = cnt[L];
      const int kn = has_next ? dc.sites[i + 1].kshard : 0;
      sa.kp_next = kn;
      sa.env_cap = ln.cap;
      sa.env_comp = h.env_comp;
      sa.slice_max = (h.m3 && !rc && !epilogue_max(h, s)) ? 1 : 0;
      sa.seed = seed;
      sa.first = lfirst;
      sa.temp = ln.temp;
      sa.alive = ln.alive;
      sa.rows_out = ln.rows;
      sa.env_next = ln.env + 2ull * h.env_comp * ln.cap * kn * h.tp_rank;
      sa.forced = forced ? ln.forced : nullptr;
      sa.marg = marg ? ln.marg : nullptr;
      sa.logscale = dc.trace ? ln.logscale : nullptr;
      sa.inv_gamma = s.inv_gamma;
      sa.trace = dc.trace ? dc.trace + i : nullptr;
      sa.scaling = h.policy.scaling;
      sa.grid = h.grid;
      sa.mu = fuse_displace ? ln.mu : nullptr;
      sa.live = dc.live + i;
      sa.near = forced ? nullptr : dc.near + i;
      sa.cinfo = cinfo;
      sa.perm = rc_pass ? ln.perm : nullptr;
      sa.rowk = rc ? ln.rowk : nullptr;
      sa.scale_out = ln.scale;
      sa.bcount = ln.bcount;
      if (rc) CUDA_OK(cudaMemsetAsync(ln.bcount, 0, 2 * (h.d + 1) * sizeof(int), ln.stream));
      launch_select(sa, ln.stream);
      if (dc.slots && active == 2 && L == 0) CUDA_OK(cudaEventRecord(ln.seldone, ln.stream));
      if (!(rc && has_next)) release_slot();
      if (rc && has_next) {
        // bucket the rows by outcome, zero the rows dead from here on, recompute the chosen slices
        PermuteArgs pa;
        pa.rows = rows[L];
        pa.d = static_cast<int>(h.d);
        pa.planes = 2 * h.env_comp;
        pa.kp = s.kshard;
        pa.env_cap = ln.cap;
        pa.rowk = ln.rowk;
        pa.scale = ln.scale;
        pa.perm = ln.perm;
        pa.env = ln.env;
        pa.bcount = ln.bcount;
        pa.bfill = ln.bcount + (h.d + 1);
        pa.rowk2 = nullptr;
        pa.scale2 = ln.scale2;
        pa.perm2 = ln.perm2;
        pa.alive2 = ln.alive2;
        pa.env2 = ln.env_perm;
        launch_permute_rows(pa, ln.stream);
        launch_zero_dead(ln.env, 2 * h.env_comp, ln.cap, kn, rows[L], ln.bcount, static_cast<int>(h.d), ln.stream);
        if (timing >= 2) CUDA_OK(cudaEventRecord(ln.gev[4 * i + 2], ln.stream));
        launch_contraction(h, dc, s, ln, i, rows[L], tma_g128, *tma_g64, cinfo, ln.stream, 2, kn);
        if (timing >= 2) CUDA_OK(cudaEventRecord(ln.gev[4 * i + 3], ln.stream));
        release_slot();
        std::swap(ln.perm, ln.perm2);
        std::swap(ln.alive, ln.alive2);
        po.launches += 4;
        po.issued += 6ull * (rows[L] + static_cast<uint64_t>(kBM) * h.d) * s.chirp * s.kp * (h.precise ? 3 : h.split ? 2 : 1);
      } else if (timing >= 2) {
        CUDA_OK(cudaEventRecord(ln.gev[4 * i + 2], ln.stream));
        CUDA_OK(cudaEventRecord(ln.gev[4 * i + 3], ln.stream));
      }
      if (xchg(h) && has_next) {  // rebuild the full environment from the column shards
        const size_t plane_b = 1ull * ln.cap * kn * sizeof(__half);
        const size_t shard_b = 2ull * h.env_comp * plane_b;
        if (h.m3) {  // ship hi / lo of re, im (planes 0, 1 and 3, 4); re-form the s planes after
          h.comm->allgather_runs(ln.env, shard_b, {{0, 2 * plane_b}, {3 * plane_b, 2 * plane_b}}, ln.stream, L);
          launch_env_reform_s(ln.env, ln.cap, kn, h.tp, rows[L], ln.stream);
          po.launches += 1;
        } else {
          h.comm->allgather(ln.env, shard_b, ln.stream, L);
        }
      }
      po.launches += 2;
      po.macs += static_cast<uint64_t>(cnt[L]) * s.chil * s.width * h.d;
      if (displaced) po.dmacs += static_cast<uint64_t>(cnt[L]) * s.width * h.d * h.d;
      po.issued += (h.m3 ? 6ull : 8ull) * rows[L] * s.np * s.kp * (h.precise ? 3 : h.split ? 2 : 1);
    }
    if (timing) CUDA_OK(cudaEventRecord(dc.ev[i + 1], dc.stream));
  }
  if (active == 2) {  // join lane 1 into lane 0
    CUDA_OK(cudaEventRecord(dc.lanes[1].done, dc.lanes[1].stream));
    CUDA_OK(cudaStreamWaitEvent(dc.stream, dc.lanes[1].done, 0));
  }
  if (timing) CUDA_OK(cudaEventRecord(dc.pass_end, dc.stream));
  CUDA_OK(cudaGetLastError());
}

struct RangeResult {
  PassOut po;
  std::vector<double> site_ms;
  std::exception_ptr err;
};

// Samples [first, first+count) on one device; rows_host may be null when rows_dev_out is set.
static void run_range(mpsg_handle_s& h, DevCtx& dc, uint64_t seed, uint64_t first,
                      uint64_t count, uint8_t* rows_host, uint8_t* rows_dev_out,
                      const uint8_t* forced_host, double* marg_host, const double* mu_host,
                      RangeResult& rr) {
  try {
    CUDA_OK(cudaSetDevice(dc.device));
    const int timing = h.opts.record_site_times;
    if (timing && dc.ev.empty()) {
      dc.ev.resize(h.M + 1);
      for (auto& e : dc.ev) CUDA_OK(cudaEventCreate(&e));
      CUDA_OK(cudaEventCreate(&dc.pass_end));
    }
    if (timing >= 2)
      for (auto& ln : dc.lanes)
        if (ln.gev.empty()) {
          ln.gev.resize(4 * h.M);
          for (auto& e : ln.gev) CUDA_OK(cudaEventCreate(&e));
        }
    if (timing) rr.site_ms.assign(h.M, 0.0);
    if (h.opts.record_decay_trace) {  // record_decay_trace
      if (!dc.trace) {
        CUDA_OK(cudaMalloc(&dc.trace, h.M * sizeof(double)));
        for (auto& ln : dc.lanes) CUDA_OK(cudaMalloc(&ln.logscale, ln.cap * sizeof(double)));
      }
      CUDA_OK(cudaMemsetAsync(dc.trace, 0, h.M * sizeof(double), dc.stream));
      CUDA_OK(cudaStreamSynchronize(dc.stream));
    }
    if (mu_host)
      for (auto& ln : dc.lanes)
        if (!ln.mu) CUDA_OK(cudaMalloc(&ln.mu, sizeof(double2) * ln.cap * h.M));
    if (!dc.live) CUDA_OK(cudaMalloc(&dc.live, h.M * sizeof(unsigned long long)));
    if (!dc.near) CUDA_OK(cudaMalloc(&dc.near, h.M * sizeof(unsigned long long)));
    CUDA_OK(cudaMemsetAsync(dc.live, 0, h.M * sizeof(unsigned long long), dc.stream));
    CUDA_OK(cudaMemsetAsync(dc.near, 0, h.M * sizeof(unsigned long long), dc.stream));
    CUDA_OK(cudaStreamSynchronize(dc.stream));
    if (forced_host || marg_host)
      for (auto& ln : dc.lanes)
        if (!ln.forced) {
          CUDA_OK(cudaMalloc(&ln.forced, 1ull * ln.cap * h.M));
          CUDA_OK(cudaMalloc(&ln.marg, 1ull * ln.cap * h.M * h.d * sizeof(double)));
        }
    for (uint64_t poff = 0; poff < count; poff += dc.cap) {
      const int n = static_cast<int>(std::min<uint64_t>(dc.cap, count - poff));
      int off[2], cnt[2];
      // the lane split is recomputed inside run_pass; forced rows must be staged first
      {
        int tmp_off[2], tmp_cnt[2];
        tmp_off[0] = 0;
        tmp_cnt[0] = n;
        tmp_cnt[1] = 0;
        if (dc.lanes.size() == 2 && n > 2 * kBM) {
          tmp_cnt[0] = std::min(dc.lanes[0].cap, round_up((n + 1) / 2, 2 * kBM));
          tmp_cnt[1] = n - tmp_cnt[0];
        }
        tmp_off[1] = tmp_cnt[0];
        if (forced_host)
          for (int L = 0; L < 2; ++L)
            if (tmp_cnt[L] > 0)
              CUDA_OK(cudaMemcpyAsync(dc.lanes[L].forced, forced_host + (poff + tmp_off[L]) * h.M,
                                      1ull * tmp_cnt[L] * h.M, cudaMemcpyHostToDevice, dc.lanes[L].stream));
        if (mu_host)
          for (int L = 0; L < 2; ++L)
            if (tmp_cnt[L] > 0)
              CUDA_OK(cudaMemcpyAsync(dc.lanes[L].mu, mu_host + 2 * (poff + tmp_off[L]) * h.M,
                                      sizeof(double2) * tmp_cnt[L] * h.M, cudaMemcpyHostToDevice,
                                      dc.lanes[L].stream));
      }
      if (timing) CUDA_OK(cudaEventRecord(dc.ev[0], dc.stream));
      run_pass(h, dc, seed, first + poff, n, forced_host != nullptr, marg_host != nullptr, mu_host != nullptr,
               rr.po, timing,
               off, cnt);
      for (int L = 0; L < 2; ++L) {
        if (cnt[L] <= 0) continue;
        Lane& ln = dc.lanes[L];
        const size_t o = (poff + off[L]) * h.M;
        if (rows_dev_out)
          CUDA_OK(cudaMemcpyAsync(rows_dev_out + o, ln.rows, 1ull * cnt[L] * h.M, cudaMemcpyDeviceToDevice,
                                  ln.stream));
        if (rows_host)
          CUDA_OK(cudaMemcpyAsync(ln.host_rows, ln.rows, 1ull * cnt[L] * h.M, cudaMemcpyDeviceToHost,
                                  ln.stream));
        if (marg_host)
          CUDA_OK(cudaMemcpyAsync(marg_host + o * h.d, ln.marg, 1ull * cnt[L] * h.M * h.d * sizeof(double),
                                  cudaMemcpyDeviceToHost, ln.stream));
      }
      for (int L = 0; L < 2; ++L)
        if (cnt[L] > 0) CUDA_OK(cudaStreamSynchronize(dc.lanes[L].stream));
      if (rows_host)
        for (int L = 0; L < 2; ++L)
          if (cnt[L] > 0)
            std::memcpy(rows_host + (poff + off[L]) * h.M, dc.lanes[L].host_rows, 1ull * cnt[L] * h.M);
      if (timing) {
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, dc.ev[0], dc.pass_end));
        rr.po.device_s += ms * 1e-3;
        for (uint64_t i = 0; i < h.M; ++i) {
          CUDA_OK(cudaEventElapsedTime(&ms, dc.ev[i], dc.ev[i + 1]));
          rr.site_ms[i] += ms;
          if (timing >= 2)
            for (int L = 0; L < 2; ++L) {
              if (cnt[L] <= 0) continue;
              CUDA_OK(cudaEventElapsedTime(&ms, dc.lanes[L].gev[4 * i], dc.lanes[L].gev[4 * i + 1]));
              rr.po.gemm_s += ms * 1e-3;
              CUDA_OK(cudaEventElapsedTime(&ms, dc.lanes[L].gev[4 * i + 2], dc.lanes[L].gev[4 * i + 3]));
              rr.po.gemm_s += ms * 1e-3;  // the slice GEMM (0 at temp-path sites)
            }
        }
      }
    }
    if (h.generated || h.file) {  // the supplied sites' finiteness / range checks (compression kernels)
      CUDA_OK(cudaStreamSynchronize(dc.copy_stream));
      check_err_flag(dc, dc.stream, h.file ? "a site streamed from the file" : "a regenerated site");
    }
    // measure's counters over the live samples (sampler.cpp:81-93,114-115)
    std::vector<unsigned long long> live(h.M);
    CUDA_OK(cudaMemcpy(live.data(), dc.live, h.M * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < h.M; ++i) {
      rr.po.wmacs += live[i] * static_cast<uint64_t>(dc.sites[i].width) * h.d;
      rr.po.pops += live[i] * h.d;
    }
    CUDA_OK(cudaMemcpy(live.data(), dc.near, h.M * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < h.M; ++i) rr.po.near += live[i];
  } catch (...) {
    rr.err = std::current_exception();
  }
}

static void sample_impl(mpsg_handle_s& h, uint64_t seed, uint64_t first, uint64_t count,
                        uint8_t* rows_host, uint8_t* rows_dev, const uint8_t* forced,
                        double* marg, mpsg_stats* st, const double* mu = nullptr) {
  config_check(mu == nullptr || h.d <= static_cast<uint64_t>(kMaxDisplacedDim),
               "displacement: phys_dim must be <= 16");
  config_check(h.finished, "state not finished (mpsg_builder_finish)");
  config_check(h.tp == 1 || h.comm != nullptr, "tensor-parallel handle not connected (mpsg_tp_connect_*)");
  config_check(h.tp == 1 || h.devs.size() == 1, "a tensor-parallel rank drives exactly one device");
  std::lock_guard<std::mutex> lk(h.mu);
  const auto t0 = std::chrono::steady_clock::now();
  const size_t nd = rows_dev ? 1 : h.devs.size();
  // devices that get no samples this call must not contribute an earlier call's trace
  for (auto& dc : h.devs)
    if (dc.trace) {
      CUDA_OK(cudaSetDevice(dc.device));
      CUDA_OK(cudaMemset(dc.trace, 0, h.M * sizeof(double)));
    }
  std::vector<RangeResult> rr(nd);
  std::vector<std::thread> th;
  for (size_t k = 0; k < nd; ++k) {
    const uint64_t a = count * k / nd, b = count * (k + 1) / nd;
    if (b <= a) continue;
    auto body = [&, k, a, b] {
      run_range(h, h.devs[k], seed, first + a, b - a, rows_host ? rows_host + a * h.M : nullptr,
                rows_dev ? rows_dev + a * h.M : nullptr, forced ? forced + a * h.M : nullptr,
                marg ? marg + a * h.M * h.d : nullptr, mu ? mu + 2 * a * h.M : nullptr, rr[k]);
    };
    if (nd == 1)
      body();
    else
      th.emplace_back(body);
  }
  for (auto& t : th) t.join();
  for (auto& r : rr)
    if (r.err) std::rethrow_exception(r.err);
  if (st) {
    st->contraction_macs = st->measure_weight_macs = st->issued_mma_flops = 0;
    st->displacement_macs = st->measure_pipeline_ops = 0;
    st->near_boundary_draws = 0;
    st->kernel_launches = 0;
    st->gemm_seconds = 0.0;
    st->device_seconds = 0.0;
    for (auto& r : rr) {
      st->contraction_macs += r.po.macs;
      st->measure_weight_macs += r.po.wmacs;
      st->displacement_macs += r.po.dmacs;
      st->measure_pipeline_ops += r.po.pops;
      st->near_boundary_draws += r.po.near;
      st->issued_mma_flops += r.po.issued;
      st->kernel_launches += r.po.launches;
      st->gemm_seconds = std::max(st->gemm_seconds, r.po.gemm_s);  // devices run concurrently
      st->device_seconds = std::max(st->device_seconds, r.po.device_s);
    }
    st->gemm_flops = 8 * st->contraction_macs;
    st->dead_samples = 0;
    if (rows_host)
      for (uint64_t n = 0; n < count; ++n) st->dead_samples += rows_host[n * h.M + h.M - 1] == kDead;
    st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    st->h2d_bytes = forced ? count * h.M : 0;
    for (auto& dc : h.devs) st->h2d_bytes += dc.h2d_bytes;
    for (auto& dc : h.devs) dc.h2d_bytes = 0;
    st->d2h_bytes = rows_host ? count * h.M : 0;
    if (st->decay_trace && h.opts.record_decay_trace) {  // sampler.cpp:196-201 normalisation
      std::vector<double> sum(h.M, 0.0), part(h.M);
      for (auto& dc : h.devs) {
        if (!dc.trace) continue;
        CUDA_OK(cudaSetDevice(dc.device));
        CUDA_OK(cudaMemcpy(part.data(), dc.trace, h.M * sizeof(double), cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < h.M; ++i) sum[i] += part[i];
      }
      for (uint64_t i = 0; i < h.M; ++i)
        st->decay_trace[i] = sum[i] / (static_cast<double>(count) * static_cast<double>(h.bonds[i + 1]));
    }
    if (st->site_seconds) {
      for (uint64_t i = 0; i < h.M; ++i) {
        double mx = 0.0;  // devices run concurrently: report the slowest
        for (auto& r : rr)
          if (!r.site_ms.empty()) mx = std::max(mx, r.site_ms[i] * 1e-3);
        st->site_seconds[i] = mx;
      }
    }
  }
}

// Teacher-forced outcomes index temp: every entry must be an outcome (< d) or the dead sentinel.
static void check_forced(const mpsg_handle_s& h, const uint8_t* forced, uint64_t count) {
  const uint64_t n = count * h.M;
  for (uint64_t j = 0; j < n; ++j)
    if (forced[j] >= h.d && forced[j] != kDead)
      throw Error(MPSG_ERR_CONFIG, "forced outcome " + std::to_string(forced[j]) + " at (sample " +
                                       std::to_string(j / h.M) + ", site " + std::to_string(j % h.M) +
                                       ") is neither < d nor the dead sentinel 0xFF");
}

void handle_chain(mpsg_handle h, uint64_t& m, uint64_t& d, std::vector<uint64_t>& bonds,
                  std::vector<const double*>& lambdas) {
  config_check(h->finished, "state not finished");
  m = h->M;
  d = h->d;
  bonds = h->bonds;
  lambdas.clear();
  for (auto& l : h->lambda) lambdas.push_back(l.data());
}

int handle_tp_size(mpsg_handle h) { return h ? h->tp : 1; }

// exchanged (weight, max) partials [tp][cap][d] per lane, allocated when the group is connected
static void ensure_part_buffers(mpsg_handle_s& h) {
  for (auto& dc : h.devs) {
    CUDA_OK(cudaSetDevice(dc.device));
    for (auto& ln : dc.lanes)
      if (!ln.part) CUDA_OK(cudaMalloc(&ln.part, 1ull * h.tp * ln.cap * h.d * sizeof(float2)));
  }
}

}  // namespace mpsg

// =============================================================================================
// C ABI
// =============================================================================================
using namespace mpsg;

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return MPSG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("out of memory: ") + e.what();
    return MPSG_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MPSG_ERR_INTERNAL;
  }
}

extern "C" {
#pragma GCC visibility push(default)

int mpsg_abi_version(void) { return MPSG_ABI_VERSION; }
const char* mpsg_last_error(void) { return g_last_error.c_str(); }

int mpsg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int c = 0;
  for (int i = 0; i < n; ++i) {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, i) == cudaSuccess &&
        major == 10)
      ++c;
  }
  return c;
}

static int begin_impl(uint64_t num_sites, uint64_t phys_dim, const uint64_t* bond_dims,
                      const mpsg_policy* policy, const mpsg_options* opts, const int* devices,
                      int ndev, mpsg_handle* out, bool generated, uint64_t gen_seed,
                      const FileMeta* fmeta = nullptr) {
  return guarded([&] {
    config_check(out != nullptr, "null output handle");
    *out = nullptr;
    validate_shape(num_sites, phys_dim, bond_dims);
    mpsg_policy pol{MPSG_F64, MPSG_F64, MPSG_SCALE_NONE};
    if (policy) pol = *policy;
    validate_policy(pol);
    auto h = std::make_unique<mpsg_handle_s>();
    h->M = num_sites;
    h->d = phys_dim;
    h->bonds.assign(bond_dims, bond_dims + num_sites + 1);
    h->policy = pol;
    if (opts) h->opts = *opts;
    config_check(h->opts.mode >= MPSG_MODE_AUTO && h->opts.mode <= MPSG_MODE_GRID, "unknown mode");
    h->precise = h->opts.mode == MPSG_MODE_PRECISE;
    h->generated = generated;
    h->gen_seed = gen_seed;
    h->file = fmeta != nullptr;
    if (fmeta) h->fmeta = *fmeta;
    if (generated || h->file) {  // regenerated / streamed into a ring of device slots (default 3)
      config_check(h->opts.host_stream_slots >= 0, "host_stream_slots must be >= 0");
      h->opts.host_stream_slots = h->opts.host_stream_slots == 0 ? 3 : std::max(2, h->opts.host_stream_slots);
    }
    {
      const char* v = std::getenv("MPSG_GEMM");  // A/B switch for the contraction kernel
      h->pair = !(v && std::string(v) == "cluster");
    }
    h->tp = std::max(1, h->opts.tp_size);
    config_check(!(h->opts.record_decay_trace && h->opts.tp_size > 1), "decay trace is not available with tensor parallelism");
    h->tp_rank = h->opts.tp_rank;
    config_check(h->tp_rank >= 0 && h->tp_rank < h->tp, "tp_rank out of range");
    config_check(h->tp == 1 || ndev <= 1, "a tensor-parallel rank drives exactly one device");
    // MPSG_MODE_GRID: the reference's TF32 / F16 compute policies on their own operand grids.  AUTO
    // picks it for those policies wherever it applies (not: generated chains, tensor parallelism,
    // the micro-batch-dependent GlobalMax scaling, the decay trace), else SINGLE.
    {
      const bool reduced = pol.compute == MPSG_TF32 || pol.compute == MPSG_F16;
      const bool applies = !generated && h->tp == 1 && pol.scaling != MPSG_SCALE_GLOBAL_MAX &&
                           !h->opts.record_decay_trace;
      if (h->opts.mode == MPSG_MODE_GRID) {
        config_check(reduced, "MPSG_MODE_GRID reproduces the TF32 / F16 compute policies (policy.compute)");
        config_check(applies, "MPSG_MODE_GRID: not with generated chains, tensor parallelism, GlobalMax "
                              "scaling or the decay trace");
      }
      if (reduced && applies && (h->opts.mode == MPSG_MODE_GRID || h->opts.mode == MPSG_MODE_AUTO))
        h->grid = pol.compute == MPSG_F16 ? kGridF16 : kGridTF32;
    }
    h->split = !h->grid && (h->opts.mode == MPSG_MODE_SPLIT || h->opts.mode == MPSG_MODE_PRECISE ||
               (h->opts.mode == MPSG_MODE_AUTO && (pol.compute == MPSG_F64 || pol.compute == MPSG_F32)));
    // the reference's F64 / F32 compute samples the caller's Gamma: AUTO keeps it to ~2^-23 (PRECISE)
    // whenever that state fits, else the fp16 format's decoded-Gamma contract (SPLIT)
    h->precise_auto = h->opts.mode == MPSG_MODE_AUTO && !generated && h->split;
    config_check(h->opts.scheme == MPSG_SCHEME_AUTO || h->opts.scheme == MPSG_SCHEME_3M ||
                     h->opts.scheme == MPSG_SCHEME_4M, "unknown contraction scheme");
    config_check(h->opts.slice >= MPSG_SLICE_AUTO && h->opts.slice <= MPSG_SLICE_RECOMPUTE,
                 "unknown slice option");
    h->gl.resize(num_sites);
    h->gr.resize(num_sites);
    for (uint64_t i = 0; i < num_sites; ++i) {
      h->gl[i].assign(h->bonds[i], 1.0);
      h->gr[i].assign(h->bonds[i + 1], 1.0);
    }
    h->site_set.assign(num_sites, 0);
    h->lambda.resize(num_sites);
    if (ndev <= 0 || devices == nullptr) {
      h->devs.resize(1);
      h->devs[0].device = 0;
    } else {
      h->devs.resize(ndev);
      for (int k = 0; k < ndev; ++k) h->devs[k].device = devices[k];
    }
    if (mpsg_device_count() == 0) throw Error(MPSG_ERR_CUDA, "no sm_100 CUDA device visible");
    choose_scheme(*h);
    h->slice_rc = h->m3 && h->tp == 1 && h->d <= 32 && h->opts.slice == MPSG_SLICE_RECOMPUTE;
    try {
      for (auto& dc : h->devs) alloc_device(*h, dc);
    } catch (...) {
      for (auto& dc : h->devs) free_device(dc);
      throw;
    }
    *out = h.release();
  });
}

int mpsg_builder_begin(uint64_t num_sites, uint64_t phys_dim, const uint64_t* bond_dims,
                       const mpsg_policy* policy, const mpsg_options* opts, const int* devices,
                       int ndev, mpsg_handle* out) {
  return begin_impl(num_sites, phys_dim, bond_dims, policy, opts, devices, ndev, out, false, 0);
}

int mpsg_generated_begin(uint64_t num_sites, uint64_t phys_dim, const uint64_t* bond_dims,
                         const mpsg_policy* policy, const mpsg_options* opts, const int* devices,
                         int ndev, uint64_t seed, mpsg_handle* out) {
  return begin_impl(num_sites, phys_dim, bond_dims, policy, opts, devices, ndev, out, true, seed);
}

int mpsg_generated_add_base(mpsg_handle h, const void* base, int base_is_device, uint64_t rows,
                            uint64_t cols, int* base_id) {
  return guarded([&] {
    config_check(h != nullptr && base != nullptr && base_id != nullptr, "null argument");
    config_check(h->generated, "not a generated handle (mpsg_generated_begin)");
    config_check(!h->finished, "builder already finished");
    config_check(rows >= 1 && cols >= 1, "empty base isometry");
    const size_t bytes = sizeof(float2) * rows * cols;
    for (size_t di = 0; di < h->devs.size(); ++di) {
      DevCtx& dc = h->devs[di];
      CUDA_OK(cudaSetDevice(dc.device));
      float2* p = nullptr;
      CUDA_OK(cudaMalloc(&p, bytes));
      dc.bases.push_back(p);
      dc.base_rows.push_back(static_cast<long long>(rows));
      dc.base_cols.push_back(static_cast<long long>(cols));
      if (!base_is_device)
        CUDA_OK(cudaMemcpy(p, base, bytes, cudaMemcpyHostToDevice));
      else if (di == 0)
        CUDA_OK(cudaMemcpy(p, base, bytes, cudaMemcpyDeviceToDevice));
      else
        CUDA_OK(cudaMemcpyPeer(p, dc.device, base, h->devs[0].device, bytes));
    }
    *base_id = static_cast<int>(h->devs[0].bases.size()) - 1;
  });
}

int mpsg_generated_set_site(mpsg_handle h, uint64_t site, int base_id, const double* lambda) {
  return guarded([&] {
    config_check(h != nullptr, "null handle");
    set_site_generated(*h, site, base_id, lambda);
  });
}

int mpsg_synthetic_site(const void* base, uint64_t ld, uint64_t rows, uint64_t cols, uint64_t phys_dim,
                        const double* lambda_prev, const double* lambda, uint64_t seed, uint64_t site,
                        void* out) {
  return guarded([&] {
    config_check(base != nullptr && lambda != nullptr && out != nullptr, "null argument");
    config_check(phys_dim >= 1 && cols % phys_dim == 0 && ld >= cols && rows >= 1, "bad generator shape");
    if (mpsg_device_count() == 0) throw Error(MPSG_ERR_CUDA, "no sm_100 CUDA device visible");
    const uint64_t chir = cols / phys_dim;
    std::vector<float> lp(rows, 1.0f), il(chir);
    if (lambda_prev)
      for (uint64_t l = 0; l < rows; ++l) lp[l] = static_cast<float>(lambda_prev[l]);
    for (uint64_t r = 0; r < chir; ++r) il[r] = 1.0f / static_cast<float>(lambda[r]);
    float *d_lp = nullptr, *d_il = nullptr;
    float2* d_ph = nullptr;
    auto cleanup = [&] {
      cudaFree(d_lp);
      cudaFree(d_il);
      cudaFree(d_ph);
    };
    try {
      CUDA_OK(cudaMalloc(&d_lp, sizeof(float) * rows));
      CUDA_OK(cudaMalloc(&d_il, sizeof(float) * chir));
      CUDA_OK(cudaMalloc(&d_ph, sizeof(float2) * cols));
      CUDA_OK(cudaMemcpy(d_lp, lp.data(), sizeof(float) * rows, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(d_il, il.data(), sizeof(float) * chir, cudaMemcpyHostToDevice));
      SynthSite g;
      g.base = static_cast<const float2*>(base);
      g.ld = static_cast<long long>(ld);
      g.cols = static_cast<long long>(cols);
      g.phase = d_ph;
      g.lam_prev = d_lp;
      g.inv_lam = d_il;
      g.d = static_cast<int>(phys_dim);
      launch_synth_phase(seed, site, static_cast<int>(cols), d_ph, nullptr);
      launch_synth_values(g, static_cast<int>(rows), static_cast<float2*>(out), nullptr);
      CUDA_OK(cudaGetLastError());
      CUDA_OK(cudaDeviceSynchronize());
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int mpsg_generated_site_values(mpsg_handle h, uint64_t site, double* out) {
  return guarded([&] {
    config_check(h != nullptr && out != nullptr, "null argument");
    config_check(h->generated, "not a generated handle (mpsg_generated_begin)");
    config_check(site < h->M && h->site_set[site], "site not set");
    std::lock_guard<std::mutex> lk(h->mu);
    DevCtx& dc = h->devs[0];
    CUDA_OK(cudaSetDevice(dc.device));
    const SiteDev& s = dc.sites[site];
    const size_t n = static_cast<size_t>(s.chil) * s.chir * h->d;
    float2* buf = nullptr;
    CUDA_OK(cudaMalloc(&buf, std::max<size_t>(1, n) * sizeof(float2)));
    std::vector<float2> v(n);
    cudaError_t e = cudaSuccess;
    try {
      CUDA_OK(cudaStreamSynchronize(dc.stream));  // the phase buffer is shared with the pass's loads
      CUDA_OK(cudaStreamSynchronize(dc.copy_stream));
      launch_synth_phase(h->gen_seed, site, s.chir * static_cast<int>(h->d), dc.phase, dc.stream);
      SynthSite g = synth_of(*h, dc, site);
      launch_synth_values(g, s.chil, buf, dc.stream);
      CUDA_OK(cudaGetLastError());
      e = cudaMemcpyAsync(v.data(), buf, n * sizeof(float2), cudaMemcpyDeviceToHost, dc.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(dc.stream);
    } catch (...) {
      cudaFree(buf);
      throw;
    }
    cudaFree(buf);
    CUDA_OK(e);
    for (size_t j = 0; j < n; ++j) {
      out[2 * j] = static_cast<double>(v[j].x);
      out[2 * j + 1] = static_cast<double>(v[j].y);
    }
  });
}

int mpsg_builder_set_site(mpsg_handle h, uint64_t site, const void* gamma, int gamma_is_device,
                          int dtype, const double* lambda) {
  return guarded([&] {
    config_check(h != nullptr, "null handle");
    set_site(*h, site, gamma, gamma_is_device != 0, dtype, lambda);
  });
}


int mpsg_builder_finish(mpsg_handle h) {
  return guarded([&] {
    config_check(h != nullptr, "null handle");
    for (uint64_t i = 0; i < h->M; ++i)
      config_check(h->site_set[i] != 0, "site " + std::to_string(i) + " was never set");
    h->finished = true;
  });
}

int mpsg_create(const mpsg_mps_view* mps, const mpsg_policy* policy, const mpsg_options* opts,
                const int* devices, int ndev, mpsg_handle* out) {
  int rc = guarded([&] {
    config_check(mps != nullptr && out != nullptr, "null argument");
    config_check(mps->gamma != nullptr && mps->lambda != nullptr, "null gamma / lambda arrays");
  });
  if (rc) return rc;
  rc = mpsg_builder_begin(mps->num_sites, mps->phys_dim, mps->bond_dims, policy, opts, devices,
                          ndev, out);
  if (rc) return rc;
  for (uint64_t i = 0; i < mps->num_sites; ++i) {
    rc = mpsg_builder_set_site(*out, i, mps->gamma[i], 0, MPSG_F64, mps->lambda[i]);
    if (rc) {
      mpsg_destroy(*out);
      *out = nullptr;
      return rc;
    }
  }
  rc = mpsg_builder_finish(*out);
  if (rc) {
    mpsg_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

void mpsg_destroy(mpsg_handle h) {
  if (!h) return;
  for (auto& dc : h->devs) free_device(dc);
  delete h;
}

uint64_t mpsg_state_bytes(mpsg_handle h) {
  if (!h || h->devs.empty()) return 0;
  uint64_t b = 0;
  if (h->generated) {  // the generators: base isometries (complex64) held per device
    for (size_t k = 0; k < h->devs[0].bases.size(); ++k)
      b += sizeof(float2) * h->devs[0].base_rows[k] * h->devs[0].base_cols[k];
    return b;
  }
  if (h->file) {  // the Gamma bytes read from storage per pass (nothing of the state is resident)
    for (uint64_t g : h->fmeta.gbytes) b += g;
    return b;
  }
  const int planes = h->devs[0].slots ? h->hplanes : h->gplanes;
  for (const auto& s : h->devs[0].sites) b += static_cast<size_t>(planes) * s.np * s.kp * sizeof(__half);
  return b;  // host-streamed: these bytes live in pinned host memory
}

int mpsg_scheme(mpsg_handle h) { return h ? (h->m3 ? MPSG_SCHEME_3M : MPSG_SCHEME_4M) : 0; }

int mpsg_gamma_store(mpsg_handle h) {
  if (!h || h->devs.empty()) return 0;
  if (h->generated) return MPSG_STORE_GENERATED;
  if (h->file) return MPSG_STORE_FILE;
  if (h->dev_store) return MPSG_STORE_COMPACT;
  return h->devs[0].slots ? MPSG_STORE_HOST : MPSG_STORE_RESIDENT;
}

int mpsg_mode(mpsg_handle h) {
  if (!h) return 0;
  if (h->grid) return MPSG_MODE_GRID;
  return h->precise ? MPSG_MODE_PRECISE : (h->split ? MPSG_MODE_SPLIT : MPSG_MODE_SINGLE);
}

int mpsg_decoded_gamma(mpsg_handle h, uint64_t site, double* out) {
  return guarded([&] {
    config_check(h != nullptr && out != nullptr, "null argument");
    config_check(site < h->M && h->site_set[site], "site not set");
    DevCtx& dc = h->devs[0];
    CUDA_OK(cudaSetDevice(dc.device));
    const SiteDev& s = dc.sites[site];
    const size_t pe = static_cast<size_t>(s.np) * s.kp;
    std::vector<__half> g(h->gplanes * pe);
    std::vector<double> cs(std::max<size_t>(1, 1ull * s.width * h->d));
    if (h->generated || h->file) {  // supply the site into a scratch buffer (the pass ring is not touched)
      std::lock_guard<std::mutex> lk(h->mu);
      CUDA_OK(cudaStreamSynchronize(dc.copy_stream));  // loads pre-issued by the last pass share the scratch
      __half* tg = nullptr;
      float2* tc = nullptr;
      CUDA_OK(cudaMalloc(&tg, g.size() * sizeof(__half)));
      cudaError_t e = cudaMalloc(&tc, sizeof(float2) * s.np);
      if (e == cudaSuccess) {
        try {
          if (h->file) {  // read + verify the payload, compress it exactly as a pass does
            std::vector<uint8_t> raw(h->fmeta.bytes[site]);
            const int fd = ::open(h->fmeta.path.c_str(), O_RDONLY);
            if (fd < 0) throw Error(MPSG_ERR_IO, "cannot open: " + h->fmeta.path);
            try {
              read_payload(fd, h->fmeta, site, raw.data());
            } catch (...) {
              ::close(fd);
              throw;
            }
            ::close(fd);
            ensure_src(dc, h->fmeta.gbytes[site]);
            CUDA_OK(cudaMemcpy(dc.src, raw.data(), h->fmeta.gbytes[site], cudaMemcpyHostToDevice));
            CUDA_OK(cudaMemset(tg, 0, g.size() * sizeof(__half)));
            CUDA_OK(cudaMemset(tc, 0, sizeof(float2) * s.np));
            launch_compress_site(dc.src, h->fmeta.prec[site], s.chil, s.chir, static_cast<int>(h->d), s.b0,
                                 s.width, s.kp, s.chirp, s.lpos_d, s.gl_d, s.gr_d, s.wl_d, h->gplanes, tg, tc,
                                 s.cs, dc.colmax, dc.err, dc.stream, h->grid);
            check_err_flag(dc, dc.stream, "site " + std::to_string(site) + " of the file");
          } else {
            regenerate_site(*h, dc, site, tg, tc, true, dc.stream);
            check_err_flag(dc, dc.stream, "regenerated site " + std::to_string(site));
          }
          e = cudaMemcpy(g.data(), tg, g.size() * sizeof(__half), cudaMemcpyDeviceToHost);
        } catch (...) {
          cudaFree(tg);
          cudaFree(tc);
          throw;
        }
      }
      cudaFree(tg);
      cudaFree(tc);
      CUDA_OK(e);
    } else if (dc.slots) {  // stored planes [Gr, Gi] per precision half: place them at their device plane
      for (int hf = 0; hf < h->hplanes / 2; ++hf)
        CUDA_OK(cudaMemcpy(g.data() + (h->m3 ? 3 : 2) * hf * pe, s.g_host + 2 * hf * pe, 2 * pe * sizeof(__half),
                           cudaMemcpyDefault));
    } else {
      CUDA_OK(cudaMemcpy(g.data(), s.g, g.size() * sizeof(__half), cudaMemcpyDeviceToHost));
    }
    CUDA_OK(cudaMemcpy(cs.data(), s.cs, cs.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const size_t d = h->d;
    std::vector<int> lpos(s.chil);
    for (int q = 0; q < h->tp; ++q) {
      int b, e;
      part_range(s.chil, h->tp, q, b, e, kgran(*h));
      for (int l = b; l < e; ++l) lpos[l] = q * s.kshard + (l - b);
    }
    for (int l = 0; l < s.chil; ++l)
      for (int rl = 0; rl < s.width; ++rl)
        for (size_t k = 0; k < d; ++k) {
          const int r = s.b0 + rl;
          const size_t row = k * s.chirp + rl;
          const double f = static_cast<double>(static_cast<float>(cs[rl * d + k])) * h->gl[site][l] /
                           h->gr[site][r];
          const size_t o = 2 * ((static_cast<size_t>(l) * s.chir + r) * d + k);
          const size_t ire = (static_cast<size_t>(kPlaneRe) * s.np + row) * s.kp + lpos[l];
          const size_t iim = (static_cast<size_t>(kPlaneIm) * s.np + row) * s.kp + lpos[l];
          double gre = __half2float(g[ire]), gim = __half2float(g[iim]);
          if (h->precise) {  // + the lo planes (3, 4): exact fp16 residuals of the hi grid
            const size_t lo = 3ull * s.np * s.kp;
            gre += static_cast<double>(__half2float(g[lo + ire]));
            gim += static_cast<double>(__half2float(g[lo + iim]));
          }
          out[o] = gre * f;
          out[o + 1] = gim * f;
        }
  });
}

int mpsg_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    config_check(id != nullptr, "null id");
    ncclUniqueId u;
    NCCL_OK(nccl().getUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

int mpsg_tp_connect_nccl(mpsg_handle h, const uint8_t id[128]) {
  return guarded([&] {
    config_check(h != nullptr && id != nullptr, "null argument");
    // tp_size 1: a one-rank group that runs the exchange data plane through NCCL (same results)
    config_check(h->devs.size() == 1, "a tensor-parallel rank drives exactly one device");
    config_check(!h->slice_rc, "the slice-recompute path has no tensor-parallel exchange");
    CUDA_OK(cudaSetDevice(h->devs[0].device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    h->comm = std::make_unique<NcclComm>(u, h->tp, h->tp_rank);
    ensure_part_buffers(*h);
  });
}

int mpsg_tp_connect_local(mpsg_handle* hs, int n) {
  return guarded([&] {
    config_check(hs != nullptr && n >= 1, "null / empty handle list");
    auto g = std::make_shared<LocalGroup>();
    g->n = n;
    g->bufs.assign(n, nullptr);
    g->ready.resize(n);
    g->done.resize(n);
    for (int r = 0; r < n; ++r) {
      config_check(hs[r] != nullptr, "null handle");
      config_check(hs[r]->tp == n && hs[r]->tp_rank == r, "handle r must have tp_size n, tp_rank r");
      g->devices.push_back(hs[r]->devs[0].device);
      CUDA_OK(cudaSetDevice(hs[r]->devs[0].device));
      CUDA_OK(cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
    }
    for (int r = 0; r < n; ++r) {
      config_check(!hs[r]->slice_rc, "the slice-recompute path has no tensor-parallel exchange");
      hs[r]->comm = std::make_unique<LocalComm>(g, r);
      ensure_part_buffers(*hs[r]);
    }
  });
}

int mpsg_sample(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count, uint8_t* rows,
                mpsg_stats* stats) {
  return guarded([&] {
    config_check(h != nullptr, "null handle");
    config_check(count == 0 || rows != nullptr, "null rows");
    config_check(count >= 1, "batch plan: total samples must be >= 1");  // sampler.cpp:21
    sample_impl(*h, seed, first, count, rows, nullptr, nullptr, nullptr, stats);
  });
}

int mpsg_sample_device(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count,
                       uint8_t* rows_dev, mpsg_stats* stats) {
  return guarded([&] {
    config_check(h != nullptr && rows_dev != nullptr, "null argument");
    config_check(count >= 1, "batch plan: total samples must be >= 1");
    sample_impl(*h, seed, first, count, nullptr, rows_dev, nullptr, nullptr, stats);
  });
}

int mpsg_marginals(mpsg_handle h, uint64_t first, uint64_t count, const uint8_t* forced,
                   double* marg) {
  return guarded([&] {
    config_check(h != nullptr && forced != nullptr && marg != nullptr, "null argument");
    config_check(count >= 1, "count must be >= 1");
    check_forced(*h, forced, count);
    std::vector<uint8_t> rows(count * h->M);
    sample_impl(*h, 0, first, count, rows.data(), nullptr, forced, marg, nullptr);
  });
}

int mpsg_sample_displaced(mpsg_handle h, uint64_t seed, uint64_t first, uint64_t count,
                          const double* mu, uint8_t* rows, mpsg_stats* stats) {
  return guarded([&] {
    config_check(h != nullptr && rows != nullptr && mu != nullptr, "null argument");
    config_check(count >= 1, "batch plan: total samples must be >= 1");
    sample_impl(*h, seed, first, count, rows, nullptr, nullptr, nullptr, stats, mu);
  });
}

int mpsg_marginals_displaced(mpsg_handle h, uint64_t first, uint64_t count, const uint8_t* forced,
                             const double* mu, double* marg) {
  return guarded([&] {
    config_check(h != nullptr && forced != nullptr && marg != nullptr && mu != nullptr, "null argument");
    config_check(count >= 1, "count must be >= 1");
    check_forced(*h, forced, count);
    std::vector<uint8_t> rows(count * h->M);
    sample_impl(*h, 0, first, count, rows.data(), nullptr, forced, marg, nullptr, mu);
  });
}

int mpsg_displacement_matrix(double mu_re, double mu_im, uint64_t n, double* out) {
  return guarded([&] {
    config_check(out != nullptr && n >= 1 && n <= 64, "displacement matrix: 1 <= n <= 64");
    if (mpsg_device_count() == 0) throw Error(MPSG_ERR_CUDA, "no sm_100 CUDA device visible");
    double2* d = nullptr;
    CUDA_OK(cudaMalloc(&d, sizeof(double2) * n * n));
    launch_displacement_matrix(mu_re, mu_im, static_cast<int>(n), d, nullptr);
    cudaError_t e = cudaMemcpy(out, d, sizeof(double2) * n * n, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CUDA_OK(e);
  });
}

int mpsg_device_draws(uint64_t seed, uint64_t first, uint64_t count, uint64_t site, double* out) {
  return guarded([&] {
    config_check(out != nullptr, "null output");
    if (mpsg_device_count() == 0) throw Error(MPSG_ERR_CUDA, "no sm_100 CUDA device visible");
    double* d = nullptr;
    CUDA_OK(cudaMalloc(&d, sizeof(double) * std::max<uint64_t>(count, 1)));
    launch_draws(seed, first, count, site, d, nullptr);
    cudaError_t e = cudaMemcpy(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CUDA_OK(e);
  });
}

int mpsg_contract_site(mpsg_handle h, uint64_t site, const double* env, uint64_t count,
                       double* temp) {
  return guarded([&] {
    config_check(h != nullptr && env != nullptr && temp != nullptr, "null argument");
    config_check(site < h->M && h->finished, "bad site / unfinished state");
    config_check(h->tp == 1, "mpsg_contract_site: not available on a tensor-parallel handle");
    config_check(h->devs[0].slots == 0, "mpsg_contract_site: not available with a slot-streamed Gamma store (host / compact 3M)");
    DevCtx& dc = h->devs[0];
    config_check(count >= 1 && count <= static_cast<uint64_t>(dc.lanes[0].cap), "count exceeds pass capacity");
    CUDA_OK(cudaSetDevice(dc.device));
    std::lock_guard<std::mutex> lk(h->mu);
    const SiteDev& s = dc.sites[site];
    const int n = static_cast<int>(count);
    const int rows = round_up(n, (h->pair && !h->m3) ? 2 * kBM : kBM);
    // host: internal env E = env * gl * sigma_n (sigma_n power of two), hi/lo fp16 planes per
    // component (re, im and, for 3M, re + im rounded once in fp32)
    Lane& ln = dc.lanes[0];
    const size_t plane = 1ull * ln.cap * s.kp;
    const int C = h->env_comp;
    std::vector<__half> e(2ull * C * plane, __float2half_rn(0.f));
    std::vector<double> sig(n, 1.0);
    for (int r = 0; r < n; ++r) {
      double mx = 0.0;
      for (int l = 0; l < s.chil; ++l) {
        const double* v = env + 2 * (static_cast<size_t>(r) * s.chil + l);
        mx = std::max(mx, std::max(std::fabs(v[0]), std::fabs(v[1])) * h->gl[site][l]);
      }
      int ex = 0;
      if (mx > 0.0) std::frexp(mx, &ex);
      sig[r] = h->grid == kGridF16 ? 1.0 : std::ldexp(1.0, kEnvExp - ex);  // the F16 grid is absolute
      for (int l = 0; l < s.chil; ++l) {
        const double* v = env + 2 * (static_cast<size_t>(r) * s.chil + l);
        __half hv[3], lv[3];
        env_split(static_cast<float>(v[0] * h->gl[site][l] * sig[r]),
                  static_cast<float>(v[1] * h->gl[site][l] * sig[r]), hv, lv);
        if (h->grid) {  // the policy's grid: RNE straight from f64, single precision half
          hv[0] = __double2half(v[0] * h->gl[site][l] * sig[r]);
          hv[1] = __double2half(v[1] * h->gl[site][l] * sig[r]);
          lv[0] = lv[1] = __float2half_rn(0.f);
        }
        const size_t o = static_cast<size_t>(r) * s.kp + l;
        for (int c = 0; c < C; ++c) {
          e[c * plane + o] = hv[c];
          e[(C + c) * plane + o] = lv[c];
        }
      }
    }
    CUDA_OK(cudaMemcpy(ln.env, e.data(), e.size() * sizeof(__half), cudaMemcpyHostToDevice));
    launch_contraction(*h, dc, s, ln, site, rows, &s.tma_g, s.tma_g64, s.cinfo, dc.stream);
    CUDA_OK(cudaGetLastError());
    std::vector<float2> t(1ull * n * h->d * s.chirp);
    CUDA_OK(cudaMemcpyAsync(t.data(), ln.temp, t.size() * sizeof(float2), cudaMemcpyDeviceToHost,
                            dc.stream));
    CUDA_OK(cudaStreamSynchronize(dc.stream));
    const size_t d = h->d;
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < s.chir; ++c)
        for (size_t k = 0; k < d; ++k) {
          const float2 v = t[(static_cast<size_t>(r) * d + k) * s.chirp + c];
          const double f = 1.0 / (h->gr[site][c] * sig[r]);
          const size_t o = 2 * ((static_cast<size_t>(r) * s.chir + c) * d + k);
          temp[o] = v.x * f;
          temp[o + 1] = v.y * f;
        }
  });
}

#pragma GCC visibility pop
}  // extern "C"

namespace mpsg {
int file_streamed_create(const std::string& path, uint64_t m, uint64_t d, const std::vector<uint64_t>& bonds,
                         const std::vector<int>& storage, const std::vector<uint64_t>& offsets,
                         const std::vector<uint64_t>& bytes, const std::vector<uint64_t>& checks,
                         const std::vector<std::vector<double>>& lambdas, const mpsg_policy* policy,
                         const mpsg_options* opts, const int* devices, int ndev, mpsg_handle* out) {
  FileMeta fm;
  fm.path = path;
  fm.off = offsets;
  fm.bytes = bytes;
  fm.check = checks;
  fm.prec = storage;
  fm.gbytes.resize(m);
  for (uint64_t i = 0; i < m; ++i) fm.gbytes[i] = bytes[i] - 8ull * bonds[i + 1];
  int rc = begin_impl(m, d, bonds.data(), policy, opts, devices, ndev, out, false, 0, &fm);
  if (rc) return rc;
  rc = guarded([&] {
    for (uint64_t i = 0; i < m; ++i) set_site_file(**out, i, lambdas[i].data());
    (*out)->finished = true;
  });
  if (rc) {
    mpsg_destroy(*out);
    *out = nullptr;
  }
  return rc;
}
}  // namespace mpsg
