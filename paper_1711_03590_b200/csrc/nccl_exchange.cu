// Native ghost exchange over NCCL point-to-point (NVLink 5 / NVSwitch).
// Replaces the reference GhostExchanger (ghost_exchange.cpp:300-398), whose
// transport is an in-process byte queue, with grouped ncclSend/ncclRecv on a
// dedicated communication stream:
//   start_update : pack owned interface cells (plan order) and post the
//                  sends; receives land directly in u's ghost region (plan
//                  order == ghost storage order, verified at setup);
//   finish_update: the compute stream waits for the receives;
//   compress     : ghost contributions travel back along the reversed
//                  routes and are added into the owned cells one neighbour
//                  at a time in ascending rank order (deterministic), then
//                  y's ghost region is zeroed.
// libnccl.so.2 is opened at run time so single-GPU use has no NCCL
// dependency (the process reuses torch's NCCL if it is already loaded).
#include "nccl_exchange.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>

namespace dgx
{
namespace
{
struct NcclApi
{
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl()
{
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char *name : {"libnccl.so.2", "libnccl.so"})
      {
        api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (api.h)
          break;
      }
    if (!api.h)
      return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
    api.Send = (decltype(api.Send))dlsym(api.h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(api.h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
  });
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv)
    fail(Code::runtime_error, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char *what)
{
  if (r != ncclSuccess)
    fail(Code::runtime_error,
         std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

dgx_status hook_start(void *ctx, void *v, void *s)
{
  return static_cast<Exchanger *>(ctx)->start_update(v, static_cast<cudaStream_t>(s));
}
dgx_status hook_finish(void *ctx, void *v, void *s)
{
  return static_cast<Exchanger *>(ctx)->finish_update(v, static_cast<cudaStream_t>(s));
}
dgx_status hook_compress(void *ctx, void *v, void *s)
{
  return static_cast<Exchanger *>(ctx)->compress(v, static_cast<cudaStream_t>(s));
}
} // namespace

void nccl_unique_id(void *id128)
{
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof id);
}

Exchanger::Exchanger(Operator *op, const void *id128, int n_ranks) : op_(op)
{
  cuda_check(cudaSetDevice(op->device()), "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t comm;
  nccl_check(nccl().CommInitRank(&comm, n_ranks, id, op->layout().rank), "ncclCommInitRank");
  comm_ = comm;
  cuda_check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming), "event");
  elem_ = op->precision() == 1 ? 4 : 8;
  const long long n_send = op->send_offsets().back(), n_recv = op->recv_offsets().back();
  const long long w = elem_ / 4; // buffers hold doubles; fp32 uses half of them
  send_buf_.resize((size_t)((n_send * w + 1) / 2 + 1));
  recv_buf_.resize((size_t)((std::max(n_send, n_recv) * w + 1) / 2 + 1));
  if (!op->recv_in_place())
    ghost_buf_.resize((size_t)((n_recv * w + 1) / 2 + 1));
}

Exchanger::~Exchanger()
{
  if (comm_ && nccl().CommDestroy)
    nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
  if (comm_stream_)
    cudaStreamDestroy(comm_stream_);
  if (ev_ready_)
    cudaEventDestroy(ev_ready_);
  if (ev_done_)
    cudaEventDestroy(ev_done_);
}

dgx_hooks Exchanger::hooks()
{
  dgx_hooks h;
  h.ctx = this;
  h.start_ghost_update = hook_start;
  h.finish_ghost_update = hook_finish;
  h.compress = hook_compress;
  return h;
}

namespace
{
template <typename F>
void typed(int elem, F &&f)
{
  if (elem == 8)
    f(double{});
  else
    f(float{});
}
} // namespace

// update_ghost_values (ghost_exchange.cpp:300-351): pack the plan values,
// one grouped NCCL send/recv per neighbour on the exchange stream; whole
// ghost cells land in place in the ghost region, partial (Hermite 2-layer)
// plans through a buffer and an indexed unpack.
dgx_status Exchanger::start_update(void *u, cudaStream_t s)
{
  if (in_flight_)
    fail(Code::logic_error, "update_ghost_values: update already in flight");
  const RankLayout &l = op_->layout();
  const ncclDataType_t dt = elem_ == 4 ? ncclFloat : ncclDouble;
  const auto &so = op_->send_offsets(), &ro = op_->recv_offsets();
  cuda_check(cudaEventRecord(ev_ready_, s), "event record");
  cuda_check(cudaStreamWaitEvent(comm_stream_, ev_ready_, 0), "wait");
  typed(elem_, [&](auto t) {
    using T = decltype(t);
    launch_gather_values<T>(static_cast<const T *>(u), op_->send_index().get(), so.back(),
                            reinterpret_cast<T *>(send_buf_.get()), comm_stream_);
  });
  char *ub = static_cast<char *>(u);
  char *sb = reinterpret_cast<char *>(send_buf_.get());
  char *rb = op_->recv_in_place() ? ub + l.owned_size() * elem_
                                  : reinterpret_cast<char *>(recv_buf_.get());
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (std::size_t i = 0; i < l.send.size(); ++i)
    nccl_check(nccl().Send(sb + so[i] * elem_, so[i + 1] - so[i], dt, l.send[i].neighbor,
                           static_cast<ncclComm_t>(comm_), comm_stream_),
               "ncclSend");
  for (std::size_t i = 0; i < l.recv.size(); ++i)
    nccl_check(nccl().Recv(rb + ro[i] * elem_, ro[i + 1] - ro[i], dt, l.recv[i].neighbor,
                           static_cast<ncclComm_t>(comm_), comm_stream_),
               "ncclRecv");
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  if (!op_->recv_in_place())
    typed(elem_, [&](auto t) {
      using T = decltype(t);
      launch_scatter_values<T>(static_cast<T *>(u), op_->recv_index().get(), ro.back(),
                               reinterpret_cast<const T *>(rb), comm_stream_);
    });
  cuda_check(cudaEventRecord(ev_done_, comm_stream_), "event record");
  in_flight_ = true;
  return DGX_OK;
}

dgx_status Exchanger::finish_update(void *, cudaStream_t s)
{
  if (!in_flight_)
    fail(Code::logic_error, "finish_ghost_update: no update was started on this vector");
  cuda_check(cudaStreamWaitEvent(s, ev_done_, 0), "wait");
  in_flight_ = false;
  return DGX_OK;
}

// compress (ghost_exchange.cpp:359-398): the ghost contributions travel the
// reversed update routes; accumulation in ascending neighbour rank, then the
// ghost region is zeroed.
dgx_status Exchanger::compress(void *y, cudaStream_t s)
{
  if (in_flight_)
    {
      cuda_check(cudaStreamWaitEvent(s, ev_done_, 0), "wait");
      in_flight_ = false;
    }
  const RankLayout &l = op_->layout();
  const ncclDataType_t dt = elem_ == 4 ? ncclFloat : ncclDouble;
  const auto &so = op_->send_offsets(), &ro = op_->recv_offsets();
  cuda_check(cudaEventRecord(ev_ready_, s), "event record");
  cuda_check(cudaStreamWaitEvent(comm_stream_, ev_ready_, 0), "wait");
  char *yb = static_cast<char *>(y);
  char *gb = yb + l.owned_size() * elem_;
  if (!op_->recv_in_place())
    {
      gb = reinterpret_cast<char *>(ghost_buf_.get());
      typed(elem_, [&](auto t) {
        using T = decltype(t);
        launch_gather_values<T>(static_cast<const T *>(y), op_->recv_index().get(), ro.back(),
                                reinterpret_cast<T *>(gb), comm_stream_);
      });
    }
  char *rb = reinterpret_cast<char *>(recv_buf_.get());
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (std::size_t i = 0; i < l.recv.size(); ++i)
    nccl_check(nccl().Send(gb + ro[i] * elem_, ro[i + 1] - ro[i], dt, l.recv[i].neighbor,
                           static_cast<ncclComm_t>(comm_), comm_stream_),
               "ncclSend");
  for (std::size_t i = 0; i < l.send.size(); ++i)
    nccl_check(nccl().Recv(rb + so[i] * elem_, so[i + 1] - so[i], dt, l.send[i].neighbor,
                           static_cast<ncclComm_t>(comm_), comm_stream_),
               "ncclRecv");
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  cuda_check(cudaEventRecord(ev_done_, comm_stream_), "event record");
  cuda_check(cudaStreamWaitEvent(s, ev_done_, 0), "wait");
  for (std::size_t i = 0; i < l.send.size(); ++i)
    typed(elem_, [&](auto t) {
      using T = decltype(t);
      launch_scatter_add_values<T>(static_cast<T *>(y), op_->send_index().get() + so[i],
                                   so[i + 1] - so[i],
                                   reinterpret_cast<const T *>(rb) + so[i], s);
    });
  const long long ghost_vals = l.total_size() - l.owned_size();
  if (ghost_vals > 0)
    cuda_check(cudaMemsetAsync(yb + l.owned_size() * elem_, 0, ghost_vals * elem_, s), "memset");
  return DGX_OK;
}

} // namespace dgx
