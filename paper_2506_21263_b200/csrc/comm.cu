// comm.cu — worker sync behind the C-ABI: NCCL over NVLink / NVSwitch, one process per GPU.
//
// The reference's "all-reduce" is a mean of per-worker reconstructions
// (collective.cpp:17-46), so the only data exchange of a round is an all-gather of every
// worker's compressed payload (the reconstruction then runs replicated, K = D * r, on every
// GPU) plus the broadcast of worker 0's float Q factors as everyone's next warm start
// (engine.cpp:241, 498-501). Both run on a library-owned side stream joined to the caller's
// stream by events, so a caller can keep other work (the next round's inner steps) on its
// own stream while the exchange is in flight.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch process that is
// the NCCL torch already loaded; a plain C++ host gets the system library. The library
// itself stays loadable (and every single-GPU entry point usable) without NCCL.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "dlx_internal.cuh"

namespace dlx {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        api.why = std::string("NCCL symbol missing: ") + name;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.AllGather, "ncclAllGather");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    api.ok = all;
  });
  if (!api.ok) raise(DLX_ERR_NCCL, api.why);
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess && r != ncclInProgress)
    raise(DLX_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

// Per-context communicator state (dlx_ctx::comm).
struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  cudaStream_t side = nullptr;      // the library's exchange stream
  cudaEvent_t ev_in = nullptr;      // caller stream -> side stream
  cudaEvent_t ev_gather = nullptr;  // all-gather landed
  cudaEvent_t ev_bcast = nullptr;   // warm-start broadcast landed
  bool bcast_pending = false;
  ~Comm() {
    if (comm) nccl().CommDestroy(comm);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_gather) cudaEventDestroy(ev_gather);
    if (ev_bcast) cudaEventDestroy(ev_bcast);
    if (side) cudaStreamDestroy(side);
  }
};

void destroy_comm(Comm* c) { delete c; }

static Comm& comm_of(dlx_ctx* ctx) {
  if (!ctx->comm) raise(DLX_ERR_VALIDATION, "context has no communicator (dlx_comm_init)");
  return *ctx->comm;
}

static void join_in(Comm& c, cudaStream_t s) {
  DLX_CUDA(cudaEventRecord(c.ev_in, s));
  DLX_CUDA(cudaStreamWaitEvent(c.side, c.ev_in, 0));
}

}  // namespace dlx

using namespace dlx;

extern "C" {

dlx_status dlx_comm_unique_id(void* out) {
  return guard([&] {
    if (!out) raise(DLX_ERR_VALIDATION, "null unique-id buffer");
    ncclUniqueId id;
    check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
  });
}

dlx_status dlx_comm_init(dlx_ctx* ctx, int rank, int world, const void* uid) {
  return guard([&] {
    if (!ctx || !uid) raise(DLX_ERR_VALIDATION, "null context or unique id");
    if (world < 1 || rank < 0 || rank >= world) raise(DLX_ERR_VALIDATION, "bad rank / world");
    if (ctx->comm) raise(DLX_ERR_VALIDATION, "context already has a communicator");
    DLX_CUDA(cudaSetDevice(ctx->device));
    auto* c = new Comm();
    c->rank = rank;
    c->world = world;
    try {
      // the exchange runs at high priority: its few CTAs are dispatched ahead of queued
      // bandwidth-bound grids on other streams
      int lo = 0, hi = 0;
      DLX_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      DLX_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
      DLX_CUDA(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
      DLX_CUDA(cudaEventCreateWithFlags(&c->ev_gather, cudaEventDisableTiming));
      DLX_CUDA(cudaEventCreateWithFlags(&c->ev_bcast, cudaEventDisableTiming));
      ncclUniqueId id;
      std::memcpy(&id, uid, sizeof(id));
      check_nccl(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    } catch (...) {
      delete c;
      throw;
    }
    ctx->comm = c;
  });
}

dlx_status dlx_comm_info(const dlx_ctx* ctx, int* rank, int* world) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (rank) *rank = ctx->comm ? ctx->comm->rank : 0;
    if (world) *world = ctx->comm ? ctx->comm->world : 1;
  });
}

dlx_status dlx_exchange(dlx_ctx* ctx, const uint8_t* d_payload, int64_t payload_bytes,
                        uint8_t* d_gathered, float* d_warm_q, int64_t warm_elems, int flags,
                        void* stream) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (payload_bytes < 0 || warm_elems < 0) raise(DLX_ERR_VALIDATION, "negative size");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DLX_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->comm || ctx->comm->world == 1) {  // D = 1: the payload is the gathered buffer
      if (d_gathered && d_gathered != d_payload && payload_bytes > 0)
        DLX_CUDA(cudaMemcpyAsync(d_gathered, d_payload, payload_bytes, cudaMemcpyDeviceToDevice, s));
      return;
    }
    Comm& c = comm_of(ctx);
    const NcclApi& n = nccl();
    NvtxRange nv("dlx_exchange");
    join_in(c, s);
    if (payload_bytes > 0) {
      // worker w's bytes land at [w * payload_bytes, (w + 1) * payload_bytes): worker order =
      // rank order, the order allreduce_avg sums in (collective.cpp:17-46)
      check_nccl(n.AllGather(d_payload, d_gathered, static_cast<size_t>(payload_bytes), ncclUint8,
                             c.comm, c.side), "ncclAllGather");
    }
    DLX_CUDA(cudaEventRecord(c.ev_gather, c.side));
    if (d_warm_q && warm_elems > 0) {
      check_nccl(n.Broadcast(d_warm_q, d_warm_q, static_cast<size_t>(warm_elems), ncclFloat32, 0,
                             c.comm, c.side), "ncclBroadcast");
      DLX_CUDA(cudaEventRecord(c.ev_bcast, c.side));
      c.bcast_pending = true;
    }
    DLX_CUDA(cudaStreamWaitEvent(s, c.ev_gather, 0));
    if (!(flags & DLX_EXCHANGE_BCAST_DEFERRED) && c.bcast_pending) {
      DLX_CUDA(cudaStreamWaitEvent(s, c.ev_bcast, 0));
      c.bcast_pending = false;
    }
    count_launch(0);
  });
}

dlx_status dlx_exchange_wait_warm(dlx_ctx* ctx, void* stream) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (ctx->comm && ctx->comm->bcast_pending) {
      DLX_CUDA(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), ctx->comm->ev_bcast, 0));
      ctx->comm->bcast_pending = false;
    }
  });
}

dlx_status dlx_comm_allgather(dlx_ctx* ctx, const void* d_send, int64_t bytes, void* d_recv,
                              void* stream) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DLX_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->comm || ctx->comm->world == 1) {
      if (d_recv != d_send && bytes > 0)
        DLX_CUDA(cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, s));
      return;
    }
    Comm& c = comm_of(ctx);
    join_in(c, s);
    check_nccl(nccl().AllGather(d_send, d_recv, static_cast<size_t>(bytes), ncclUint8, c.comm,
                                c.side), "ncclAllGather");
    DLX_CUDA(cudaEventRecord(c.ev_gather, c.side));
    DLX_CUDA(cudaStreamWaitEvent(s, c.ev_gather, 0));
  });
}

dlx_status dlx_comm_allreduce_sum_f64(dlx_ctx* ctx, double* d_buf, int64_t n, void* stream) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (!ctx->comm || ctx->comm->world == 1 || n == 0) return;
    Comm& c = comm_of(ctx);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DLX_CUDA(cudaSetDevice(ctx->device));
    join_in(c, s);
    check_nccl(nccl().AllReduce(d_buf, d_buf, static_cast<size_t>(n), ncclFloat64, ncclSum, c.comm,
                                c.side), "ncclAllReduce");
    DLX_CUDA(cudaEventRecord(c.ev_gather, c.side));
    DLX_CUDA(cudaStreamWaitEvent(s, c.ev_gather, 0));
  });
}

dlx_status dlx_comm_check(dlx_ctx* ctx) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (!ctx->comm) return;
    ncclResult_t r = ncclSuccess;
    check_nccl(nccl().CommGetAsyncError(ctx->comm->comm, &r), "ncclCommGetAsyncError");
    if (r != ncclSuccess && r != ncclInProgress)
      raise(DLX_ERR_NCCL, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(r));
  });
}

dlx_status dlx_comm_destroy(dlx_ctx* ctx) {
  return guard([&] {
    if (!ctx) raise(DLX_ERR_VALIDATION, "null context");
    if (ctx->comm) {
      DLX_CUDA(cudaSetDevice(ctx->device));
      DLX_CUDA(cudaStreamSynchronize(ctx->comm->side));
      delete ctx->comm;
      ctx->comm = nullptr;
    }
  });
}

}  // extern "C"
