// Exchange layer: pack kernels, NCCL transport (loaded at run time), in-process loopback transport,
// and the host-bootstrapped CUDA-IPC transport (one process per rank on devices that can map each
// other's memory, host collectives through caller callbacks, e.g. a gloo process group).
//
// Forward exchange (Alg. 1 lines 2 and 5): K||V rows of remote columns, packed
// [k | v] per row.  Backward exchange (reading Z11, transposed owner), in two messages so the first
// overlaps the row pass: [q | dy] rows of in-neighbour rows (known at backward entry), then their
// (LSE2, D) blocks (written by the row pass).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "gt_internal.h"

// ------------------------------------------------------------------ packing --
namespace gt {
namespace {

__global__ void pack_kv_kernel(const uint4* k, const uint4* v, const int32_t* idx, int64_t rows, int vec,
                               uint4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw) {
    const int64_t src = idx[r];
    uint4* o = out + r * 2 * vec;
    for (int c = lane; c < vec; c += 32) {
      o[c] = k[src * vec + c];
      o[vec + c] = v[src * vec + c];
    }
  }
}

__global__ void pack_stats_kernel(const uint4* stats, const int32_t* idx, int64_t rows, int svec, uint4* out) {
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows * svec; t += nt) {
    const int64_t r = t / svec;
    const int c = (int)(t % svec);
    out[r * svec + c] = stats[(int64_t)idx[r] * svec + c];
  }
}

// GP-A2A head-group transposes.  A row of `groups` head groups of `gb` bytes each:
//   pack:   src[row][s] -> dst[s][row] (groups s != self), dst_self[row] (s == self)
//   unpack: src[s][row] (s != self), src_self[row] (s == self) -> dst[row][s]
template <typename U>
__global__ void a2a_pack_kernel(const U* src, int64_t rows, int groups, int64_t gu, int self, U* dst, U* dst_self) {
  const int64_t total = rows * groups * gu;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % gu;
    const int64_t rs = t / gu;
    const int s = (int)(rs % groups);
    const int64_t r = rs / groups;
    const U x = src[t];
    if (s == self) dst_self[r * gu + c] = x;
    else dst[((int64_t)s * rows + r) * gu + c] = x;
  }
}
template <typename U>
__global__ void a2a_unpack_kernel(const U* src, const U* src_self, int64_t rows, int groups, int64_t gu, int self,
                                  U* dst) {
  const int64_t total = rows * groups * gu;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % gu;
    const int64_t rs = t / gu;
    const int s = (int)(rs % groups);
    const int64_t r = rs / groups;
    dst[t] = s == self ? src_self[r * gu + c] : src[((int64_t)s * rows + r) * gu + c];
  }
}

}  // namespace

gt_status a2a_pack(const void* src, int64_t rows, int groups, int64_t gb, int self, void* dst, void* dst_self,
                   cudaStream_t st) {
  if (rows <= 0) return GT_OK;
  const int64_t n = rows * groups * (gb % 16 == 0 ? gb / 16 : gb / 4);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (gb % 16 == 0)
    a2a_pack_kernel<uint4><<<blocks, 256, 0, st>>>((const uint4*)src, rows, groups, gb / 16, self, (uint4*)dst,
                                                   (uint4*)dst_self);
  else
    a2a_pack_kernel<uint32_t><<<blocks, 256, 0, st>>>((const uint32_t*)src, rows, groups, gb / 4, self,
                                                      (uint32_t*)dst, (uint32_t*)dst_self);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

gt_status a2a_unpack(const void* src, const void* src_self, int64_t rows, int groups, int64_t gb, int self, void* dst,
                     cudaStream_t st) {
  if (rows <= 0) return GT_OK;
  const int64_t n = rows * groups * (gb % 16 == 0 ? gb / 16 : gb / 4);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (gb % 16 == 0)
    a2a_unpack_kernel<uint4><<<blocks, 256, 0, st>>>((const uint4*)src, (const uint4*)src_self, rows, groups, gb / 16,
                                                     self, (uint4*)dst);
  else
    a2a_unpack_kernel<uint32_t><<<blocks, 256, 0, st>>>((const uint32_t*)src, (const uint32_t*)src_self, rows, groups,
                                                        gb / 4, self, (uint32_t*)dst);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

gt_status pack_kv(const void* k, const void* v, const int32_t* idx, int64_t rows, int64_t D, int elt, void* out,
                  cudaStream_t st) {
  if (rows <= 0) return GT_OK;
  const int vec = (int)(D * elt / 16);
  int64_t blocks = std::min<int64_t>((rows + 7) / 8, 148 * 16);
  pack_kv_kernel<<<(int)blocks, 256, 0, st>>>((const uint4*)k, (const uint4*)v, idx, rows, vec, (uint4*)out);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

gt_status pack_stats(const float* stats, const int32_t* idx, int64_t rows, int64_t row_bytes, void* out,
                     cudaStream_t st) {
  if (rows <= 0) return GT_OK;
  const int svec = (int)(row_bytes / 16);
  const int64_t blocks = std::min<int64_t>((rows * svec + 255) / 256, 148 * 8);
  pack_stats_kernel<<<(int)blocks, 256, 0, st>>>((const uint4*)stats, idx, rows, svec, (uint4*)out);
  GT_CUDA_TRY(cudaGetLastError());
  return GT_OK;
}

// -------------------------------------------------------------------- NCCL --
namespace {

typedef void* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclUint8 = 1, ncclInt32 = 2, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("GT_NCCL_LIB");
    void* h = nullptr;
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.err = "libnccl.so.2 not found (set GT_NCCL_LIB)"; return; }
#define GT_SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
    GT_SYM(GetUniqueId); GT_SYM(CommInitRank); GT_SYM(CommDestroy); GT_SYM(AllGather); GT_SYM(AllReduce);
    GT_SYM(Broadcast); GT_SYM(Send); GT_SYM(Recv); GT_SYM(GroupStart); GT_SYM(GroupEnd); GT_SYM(GetErrorString);
#undef GT_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.Send || !api.Recv || !api.GroupStart ||
        !api.GroupEnd || !api.Broadcast || !api.AllReduce) {
      api.err = "libnccl is missing required symbols";
      return;
    }
    api.loaded = true;
  });
  return api;
}

#define GT_NCCL_TRY(expr)                                                                            \
  do {                                                                                               \
    ncclResult_t _r = (expr);                                                                        \
    if (_r != 0)                                                                                     \
      return ::gt::fail(GT_ENCCL, std::string(#expr) + ": " +                                        \
                                      (nccl().GetErrorString ? nccl().GetErrorString(_r) : "error")); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t c;
  int w, r;
  DevBuf scratch;
  NcclComm(ncclComm_t c_, int w_, int r_) : c(c_), w(w_), r(r_) {}
  int world() const override { return w; }
  int rank() const override { return r; }
  gt_status exchange(const void* send_buf, const int64_t* send_off, const int64_t* send_cnt, void* recv_buf,
                     const int64_t* recv_off, const int64_t* recv_cnt, int64_t row_bytes,
                     cudaStream_t stream) override {
    NcclApi& a = nccl();
    GT_NCCL_TRY(a.GroupStart());
    for (int s = 0; s < w; ++s) {
      if (s == r) continue;
      if (send_cnt[s] > 0)
        GT_NCCL_TRY(a.Send((const char*)send_buf + send_off[s] * row_bytes, (size_t)(send_cnt[s] * row_bytes),
                           ncclUint8, s, c, stream));
      if (recv_cnt[s] > 0)
        GT_NCCL_TRY(a.Recv((char*)recv_buf + recv_off[s] * row_bytes, (size_t)(recv_cnt[s] * row_bytes), ncclUint8,
                           s, c, stream));
    }
    GT_NCCL_TRY(a.GroupEnd());
    return GT_OK;
  }
  gt_status all_gather(const void* send_buf, void* recv_buf, int64_t rows, int64_t row_bytes,
                       cudaStream_t stream) override {
    if (rows == 0) return GT_OK;
    GT_NCCL_TRY(nccl().AllGather(send_buf, recv_buf, (size_t)(rows * row_bytes), ncclUint8, c, stream));
    return GT_OK;
  }
  gt_status ensure_scratch() {
    if (!scratch.p) GT_TRY(scratch.alloc(4096));
    return GT_OK;
  }
  gt_status broadcast_host(void* data, int64_t bytes, cudaStream_t stream) override {
    GT_TRY(ensure_scratch());
    if (bytes > 4096) return fail(GT_EINVAL, "broadcast_host: too large");
    GT_CUDA_TRY(cudaMemcpyAsync(scratch.p, data, bytes, cudaMemcpyHostToDevice, stream));
    GT_NCCL_TRY(nccl().Broadcast(scratch.p, scratch.p, (size_t)bytes, ncclUint8, 0, c, stream));
    GT_CUDA_TRY(cudaMemcpyAsync(data, scratch.p, bytes, cudaMemcpyDeviceToHost, stream));
    GT_CUDA_TRY(cudaStreamSynchronize(stream));
    return GT_OK;
  }
  gt_status max_host(double* v, cudaStream_t stream) override {
    GT_TRY(ensure_scratch());
    GT_CUDA_TRY(cudaMemcpyAsync(scratch.p, v, sizeof(double), cudaMemcpyHostToDevice, stream));
    GT_NCCL_TRY(nccl().AllReduce(scratch.p, scratch.p, 1, ncclFloat64, ncclMax, c, stream));
    GT_CUDA_TRY(cudaMemcpyAsync(v, scratch.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
    GT_CUDA_TRY(cudaStreamSynchronize(stream));
    return GT_OK;
  }
  gt_status barrier(cudaStream_t stream) override {
    double x = 0;
    return max_host(&x, stream);
  }
  gt_status stream_barrier(cudaStream_t stream) override {
    // an all-reduce of one word completes on no rank before every rank has entered it
    GT_TRY(ensure_scratch());
    GT_NCCL_TRY(nccl().AllReduce((char*)scratch.p + 2048, (char*)scratch.p + 2048, 1, ncclInt32, ncclSum, c, stream));
    return GT_OK;
  }
  std::vector<void*> opened;  // IPC mappings to close
  gt_status share_pointers(void* local, void** peers, cudaStream_t stream) override {
    GT_TRY(ensure_scratch());
    if ((int64_t)sizeof(cudaIpcMemHandle_t) * w > 2048) return fail(GT_ECONFIG, "share_pointers: world too large");
    cudaIpcMemHandle_t mine;
    GT_CUDA_TRY(cudaIpcGetMemHandle(&mine, local));
    GT_CUDA_TRY(cudaMemcpyAsync((char*)scratch.p + r * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice,
                                stream));
    GT_NCCL_TRY(nccl().AllGather((char*)scratch.p + r * sizeof(mine), scratch.p, sizeof(mine), ncclUint8, c, stream));
    std::vector<cudaIpcMemHandle_t> all((size_t)w);
    GT_CUDA_TRY(cudaMemcpyAsync(all.data(), scratch.p, sizeof(mine) * w, cudaMemcpyDeviceToHost, stream));
    GT_CUDA_TRY(cudaStreamSynchronize(stream));
    for (int s = 0; s < w; ++s) {
      if (s == r) {
        peers[s] = local;
        continue;
      }
      void* p = nullptr;
      GT_CUDA_TRY(cudaIpcOpenMemHandle(&p, all[(size_t)s], cudaIpcMemLazyEnablePeerAccess));
      opened.push_back(p);
      peers[s] = p;
    }
    return GT_OK;
  }
  ~NcclComm() override {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};

}  // namespace

Comm* make_nccl_comm(void* nccl_comm, int world, int rank, gt_status* st) {
  if (!nccl().loaded) {
    *st = fail(GT_ENCCL, nccl().err);
    return nullptr;
  }
  *st = GT_OK;
  return new NcclComm((ncclComm_t)nccl_comm, world, rank);
}

}  // namespace gt

// ---------------------------------------------------------------- loopback --
struct gt_loopback_s {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  struct Slot {
    const void* send = nullptr;
    const int64_t* off = nullptr;
    const int64_t* cnt = nullptr;
    int64_t row_bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    std::vector<char> host;
    double val = 0;
    void* ptr = nullptr;
  };
  std::vector<Slot> slots;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace gt {
namespace {

struct LoopbackComm : Comm {
  gt_loopback_s* g;
  int r;
  cudaEvent_t ready = nullptr, done = nullptr;
  std::vector<int64_t> ag_off, ag_cnt, ag_roff;
  LoopbackComm(gt_loopback_s* g_, int r_) : g(g_), r(r_) {
    cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  }
  ~LoopbackComm() override {
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
  }
  int world() const override { return g->world; }
  int rank() const override { return r; }
  gt_status exchange(const void* send_buf, const int64_t* send_off, const int64_t* send_cnt, void* recv_buf,
                     const int64_t* recv_off, const int64_t* recv_cnt, int64_t row_bytes,
                     cudaStream_t stream) override {
    const int w = g->world;
    GT_CUDA_TRY(cudaEventRecord(ready, stream));
    auto& me = g->slots[r];
    me.send = send_buf; me.off = send_off; me.cnt = send_cnt; me.row_bytes = row_bytes; me.ready = ready;
    g->barrier();
    gt_status st = GT_OK;
    for (int s = 0; s < w && st == GT_OK; ++s) {
      if (s == r) continue;
      const auto& peer = g->slots[s];
      if (peer.row_bytes != row_bytes || peer.cnt[r] != recv_cnt[s]) {
        st = fail(GT_ENCCL, "loopback exchange: protocol mismatch between ranks " + std::to_string(r) + " and " +
                                std::to_string(s));
        break;
      }
      if (recv_cnt[s] == 0) continue;
      if (cudaStreamWaitEvent(stream, peer.ready, 0) != cudaSuccess ||
          cudaMemcpyAsync((char*)recv_buf + recv_off[s] * row_bytes, (const char*)peer.send + peer.off[r] * row_bytes,
                          (size_t)(recv_cnt[s] * row_bytes), cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        st = fail(GT_ECUDA, "loopback exchange: copy failed");
    }
    cudaEventRecord(done, stream);
    me.done = done;
    g->barrier();
    for (int s = 0; s < w; ++s)
      if (s != r) cudaStreamWaitEvent(stream, g->slots[s].done, 0);
    g->barrier();
    return st;
  }
  gt_status all_gather(const void* send_buf, void* recv_buf, int64_t rows, int64_t row_bytes,
                       cudaStream_t stream) override {
    const int w = g->world;
    ag_off.assign(w, 0);
    ag_cnt.assign(w, rows);
    ag_roff.resize(w);
    for (int s = 0; s < w; ++s) ag_roff[s] = s * rows;
    if (rows > 0)
      GT_CUDA_TRY(cudaMemcpyAsync((char*)recv_buf + r * rows * row_bytes, send_buf, (size_t)(rows * row_bytes),
                                  cudaMemcpyDeviceToDevice, stream));
    return exchange(send_buf, ag_off.data(), ag_cnt.data(), recv_buf, ag_roff.data(), ag_cnt.data(), row_bytes,
                    stream);
  }
  gt_status broadcast_host(void* data, int64_t bytes, cudaStream_t) override {
    if (r == 0) g->slots[0].host.assign((const char*)data, (const char*)data + bytes);
    g->barrier();
    std::memcpy(data, g->slots[0].host.data(), (size_t)bytes);
    g->barrier();
    return GT_OK;
  }
  gt_status max_host(double* v, cudaStream_t) override {
    g->slots[r].val = *v;
    g->barrier();
    double m = *v;
    for (int s = 0; s < g->world; ++s) m = std::max(m, g->slots[s].val);
    g->barrier();
    *v = m;
    return GT_OK;
  }
  gt_status barrier(cudaStream_t) override {
    g->barrier();
    return GT_OK;
  }
  gt_status stream_barrier(cudaStream_t stream) override {
    GT_CUDA_TRY(cudaEventRecord(ready, stream));
    g->slots[r].ready = ready;
    g->barrier();
    for (int s = 0; s < g->world; ++s)
      if (s != r) GT_CUDA_TRY(cudaStreamWaitEvent(stream, g->slots[s].ready, 0));
    g->barrier();  // nobody re-records its event before every rank has enqueued its waits
    return GT_OK;
  }
  gt_status share_pointers(void* local, void** peers, cudaStream_t) override {
    g->slots[r].ptr = local;
    g->barrier();
    for (int s = 0; s < g->world; ++s) peers[s] = g->slots[s].ptr;
    g->barrier();
    return GT_OK;
  }
};

}  // namespace

Comm* make_loopback_comm(gt_loopback_t g, int world, int rank, gt_status* st) {
  if (!g || g->world != world) {
    *st = fail(GT_EINVAL, "loopback group size does not match world");
    return nullptr;
  }
  *st = GT_OK;
  return new LoopbackComm(g, rank);
}

}  // namespace gt

// ----------------------------------------------------------------- host IPC --
// One process per rank.  Host collectives (an all-gather of a few bytes) go through the caller's
// callback; device data moves by CUDA IPC: each rank publishes the IPC handle of the allocation holding
// its send rows and an interprocess event recorded after they were written; the receivers wait on that
// event on their own stream and copy straight out of the mapped peer allocation (cudaMemcpyAsync
// device to device), then every rank waits on the receivers' "done" events before its send rows may be
// rewritten.  Same protocol as the loopback transport, across processes.
struct gt_hostipc_s {
  gt_host_coll coll;
  int world = 1, rank = 0, device = 0;
  cudaEvent_t ready = nullptr, done = nullptr;          // this rank's interprocess events
  std::vector<cudaEvent_t> peer_ready, peer_done;       // opened peer events (own slot: own events)
  std::map<std::string, void*> opened;                  // peer allocation (handle bytes) -> mapping
  std::mutex mu;
  ~gt_hostipc_s() {
    for (auto& kv : opened) cudaIpcCloseMemHandle(kv.second);
    for (int s = 0; s < world; ++s)
      if (s != rank) {
        if (s < (int)peer_ready.size() && peer_ready[s]) cudaEventDestroy(peer_ready[s]);
        if (s < (int)peer_done.size() && peer_done[s]) cudaEventDestroy(peer_done[s]);
      }
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
  }
  gt_status allgather(const void* send, void* recv, int64_t bytes) {
    if (coll.allgather(coll.ctx, send, recv, bytes) != 0)
      return gt::fail(GT_ENCCL, "host IPC: the host all-gather callback failed");
    return GT_OK;
  }
  gt_status barrier() {
    char x = 0;
    std::vector<char> all((size_t)world);
    return allgather(&x, all.data(), 1);
  }
};

namespace gt {
namespace {

// base of the allocation holding p and p's offset in it (cudaIpcGetMemHandle needs the base)
gt_status alloc_base(const void* p, char** base, int64_t* off) {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(f);
  });
  if (!fn) return fail(GT_ECUDA, "cuMemGetAddressRange is not available");
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return fail(GT_ECUDA, "host IPC: not a device allocation");
  *base = (char*)b;
  *off = (int64_t)((const char*)p - (const char*)b);
  return GT_OK;
}

struct IpcRef {            // one rank's published buffer
  cudaIpcMemHandle_t h;
  int64_t off;
};

gt_status publish(gt_hostipc_s* g, const void* p, std::vector<IpcRef>& all, bool has) {
  IpcRef mine;
  std::memset(&mine, 0, sizeof(mine));
  if (has) {
    char* base = nullptr;
    GT_TRY(alloc_base(p, &base, &mine.off));
    GT_CUDA_TRY(cudaIpcGetMemHandle(&mine.h, base));
  } else {
    mine.off = -1;
  }
  all.resize((size_t)g->world);
  return g->allgather(&mine, all.data(), sizeof(mine));
}

gt_status open_ref(gt_hostipc_s* g, const IpcRef& ref, char** out) {
  std::string key((const char*)&ref.h, sizeof(ref.h));
  auto it = g->opened.find(key);
  if (it == g->opened.end()) {
    void* p = nullptr;
    GT_CUDA_TRY(cudaIpcOpenMemHandle(&p, ref.h, cudaIpcMemLazyEnablePeerAccess));
    it = g->opened.emplace(key, p).first;
  }
  *out = (char*)it->second + ref.off;
  return GT_OK;
}

struct HostIpcComm : Comm {
  gt_hostipc_s* g;
  explicit HostIpcComm(gt_hostipc_s* g_) : g(g_) {}
  int world() const override { return g->world; }
  int rank() const override { return g->rank; }
  // every rank records `done` after its receives, then waits on every peer's `done` (its own send rows
  // may only be rewritten after all readers copied them); the final barrier keeps events from being
  // re-recorded before every rank has enqueued its waits
  gt_status finish(cudaStream_t stream, gt_status st) {
    if (cudaEventRecord(g->done, stream) != cudaSuccess && st == GT_OK) st = fail(GT_ECUDA, "host IPC: record");
    gt_status b = g->barrier();
    if (b != GT_OK) return b;
    for (int s = 0; s < g->world; ++s)
      if (s != g->rank && cudaStreamWaitEvent(stream, g->peer_done[s], 0) != cudaSuccess && st == GT_OK)
        st = fail(GT_ECUDA, "host IPC: wait");
    b = g->barrier();
    return b != GT_OK ? b : st;
  }
  gt_status exchange(const void* send_buf, const int64_t* send_off, const int64_t* send_cnt, void* recv_buf,
                     const int64_t* recv_off, const int64_t* recv_cnt, int64_t row_bytes,
                     cudaStream_t stream) override {
    std::lock_guard<std::mutex> lock(g->mu);
    const int w = g->world, r = g->rank;
    int64_t nsend = 0;
    for (int s = 0; s < w; ++s)
      if (s != r) nsend += send_cnt[s];
    GT_CUDA_TRY(cudaEventRecord(g->ready, stream));
    std::vector<IpcRef> refs;
    GT_TRY(publish(g, send_buf, refs, nsend > 0 && send_buf));
    // protocol record: row size and this rank's (offset, count) per destination
    std::vector<int64_t> mine(1 + 2 * (size_t)w), all((size_t)w * (1 + 2 * (size_t)w));
    mine[0] = row_bytes;
    for (int s = 0; s < w; ++s) { mine[1 + 2 * s] = send_off[s]; mine[2 + 2 * s] = send_cnt[s]; }
    GT_TRY(g->allgather(mine.data(), all.data(), (int64_t)(mine.size() * sizeof(int64_t))));
    gt_status st = GT_OK;
    for (int s = 0; s < w && st == GT_OK; ++s) {
      if (s == r) continue;
      const int64_t* pr = all.data() + (size_t)s * (1 + 2 * w);
      if (pr[0] != row_bytes || pr[2 + 2 * r] != recv_cnt[s]) {
        st = fail(GT_ENCCL, "host IPC exchange: protocol mismatch between ranks " + std::to_string(r) + " and " +
                                std::to_string(s));
        break;
      }
      if (recv_cnt[s] == 0) continue;
      char* src = nullptr;
      st = open_ref(g, refs[(size_t)s], &src);
      if (st != GT_OK) break;
      if (cudaStreamWaitEvent(stream, g->peer_ready[s], 0) != cudaSuccess ||
          cudaMemcpyAsync((char*)recv_buf + recv_off[s] * row_bytes, src + pr[1 + 2 * r] * row_bytes,
                          (size_t)(recv_cnt[s] * row_bytes), cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        st = fail(GT_ECUDA, "host IPC exchange: copy failed");
    }
    return finish(stream, st);
  }
  std::vector<int64_t> ag_off, ag_cnt, ag_roff;
  gt_status all_gather(const void* send_buf, void* recv_buf, int64_t rows, int64_t row_bytes,
                       cudaStream_t stream) override {
    const int w = g->world, r = g->rank;
    ag_off.assign(w, 0);
    ag_cnt.assign(w, rows);
    ag_roff.resize(w);
    for (int s = 0; s < w; ++s) ag_roff[s] = s * rows;
    if (rows > 0)
      GT_CUDA_TRY(cudaMemcpyAsync((char*)recv_buf + r * rows * row_bytes, send_buf, (size_t)(rows * row_bytes),
                                  cudaMemcpyDeviceToDevice, stream));
    return exchange(send_buf, ag_off.data(), ag_cnt.data(), recv_buf, ag_roff.data(), ag_cnt.data(), row_bytes,
                    stream);
  }
  gt_status broadcast_host(void* data, int64_t bytes, cudaStream_t) override {
    std::vector<char> all((size_t)(bytes * g->world));
    GT_TRY(g->allgather(data, all.data(), bytes));
    std::memcpy(data, all.data(), (size_t)bytes);  // rank 0's
    return GT_OK;
  }
  gt_status max_host(double* v, cudaStream_t) override {
    std::vector<double> all((size_t)g->world);
    GT_TRY(g->allgather(v, all.data(), sizeof(double)));
    for (double x : all) *v = std::max(*v, x);
    return GT_OK;
  }
  gt_status barrier(cudaStream_t) override { return g->barrier(); }
  gt_status stream_barrier(cudaStream_t stream) override {
    std::lock_guard<std::mutex> lock(g->mu);
    GT_CUDA_TRY(cudaEventRecord(g->ready, stream));
    GT_TRY(g->barrier());
    gt_status st = GT_OK;
    for (int s = 0; s < g->world; ++s)
      if (s != g->rank && cudaStreamWaitEvent(stream, g->peer_ready[s], 0) != cudaSuccess)
        st = fail(GT_ECUDA, "host IPC: stream barrier wait");
    GT_TRY(g->barrier());
    return st;
  }
  gt_status share_pointers(void* local, void** peers, cudaStream_t) override {
    std::lock_guard<std::mutex> lock(g->mu);
    std::vector<IpcRef> refs;
    GT_TRY(publish(g, local, refs, local != nullptr));
    for (int s = 0; s < g->world; ++s) {
      if (s == g->rank || refs[(size_t)s].off < 0) {
        peers[s] = s == g->rank ? local : nullptr;
        continue;
      }
      char* p = nullptr;
      GT_TRY(open_ref(g, refs[(size_t)s], &p));
      peers[s] = p;
    }
    return GT_OK;
  }
};

}  // namespace

Comm* make_hostipc_comm(gt_hostipc_t g, int world, int rank, gt_status* st) {
  if (!g || g->world != world || g->rank != rank) {
    *st = fail(GT_EINVAL, "host IPC group does not match (world, rank)");
    return nullptr;
  }
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != g->device) {
    *st = fail(GT_EINVAL, "host IPC group was created on another device");
    return nullptr;
  }
  *st = GT_OK;
  return new HostIpcComm(g);
}

}  // namespace gt

using namespace gt;

extern "C" {

gt_status gt_loopback_create(int world, gt_loopback_t* out) {
  if (world < 1 || !out) return fail(GT_EINVAL, "gt_loopback_create: bad arguments");
  auto* g = new gt_loopback_s();
  g->world = world;
  g->slots.resize(world);
  *out = g;
  return GT_OK;
}

void gt_loopback_destroy(gt_loopback_t g) { delete g; }

gt_status gt_hostipc_create(const gt_host_coll* coll, int world, int rank, gt_hostipc_t* out) {
  if (!coll || !coll->allgather || !out || world < 1 || rank < 0 || rank >= world)
    return fail(GT_EINVAL, "gt_hostipc_create: bad arguments");
  *out = nullptr;
  auto g = std::make_unique<gt_hostipc_s>();
  g->coll = *coll;
  g->world = world;
  g->rank = rank;
  GT_CUDA_TRY(cudaGetDevice(&g->device));
  const unsigned fl = cudaEventDisableTiming | cudaEventInterprocess;
  GT_CUDA_TRY(cudaEventCreateWithFlags(&g->ready, fl));
  GT_CUDA_TRY(cudaEventCreateWithFlags(&g->done, fl));
  cudaIpcEventHandle_t mine[2];
  GT_CUDA_TRY(cudaIpcGetEventHandle(&mine[0], g->ready));
  GT_CUDA_TRY(cudaIpcGetEventHandle(&mine[1], g->done));
  std::vector<cudaIpcEventHandle_t> all((size_t)world * 2);
  GT_TRY(g->allgather(mine, all.data(), sizeof(mine)));
  g->peer_ready.assign(world, nullptr);
  g->peer_done.assign(world, nullptr);
  for (int s = 0; s < world; ++s) {
    if (s == rank) {
      g->peer_ready[s] = g->ready;
      g->peer_done[s] = g->done;
      continue;
    }
    GT_CUDA_TRY(cudaIpcOpenEventHandle(&g->peer_ready[s], all[2 * (size_t)s]));
    GT_CUDA_TRY(cudaIpcOpenEventHandle(&g->peer_done[s], all[2 * (size_t)s + 1]));
  }
  *out = g.release();
  return GT_OK;
}

void gt_hostipc_destroy(gt_hostipc_t g) { delete g; }

gt_status gt_nccl_unique_id(void* uid128) {
  if (!uid128) return fail(GT_EINVAL, "null uid");
  if (!nccl().loaded) return fail(GT_ENCCL, nccl().err);
  ncclUniqueId id;
  GT_NCCL_TRY(nccl().GetUniqueId(&id));
  std::memcpy(uid128, &id, sizeof(id));
  return GT_OK;
}

gt_status gt_nccl_comm_create(const void* uid128, int world, int rank, void** comm) {
  if (!uid128 || !comm || world < 1 || rank < 0 || rank >= world) return fail(GT_EINVAL, "bad arguments");
  if (!nccl().loaded) return fail(GT_ENCCL, nccl().err);
  ncclUniqueId id;
  std::memcpy(&id, uid128, sizeof(id));
  ncclComm_t c = nullptr;
  GT_NCCL_TRY(nccl().CommInitRank(&c, world, id, rank));
  *comm = c;
  return GT_OK;
}

void gt_nccl_comm_destroy(void* comm) {
  if (comm && nccl().loaded && nccl().CommDestroy) nccl().CommDestroy((ncclComm_t)comm);
}

}  // extern "C"
