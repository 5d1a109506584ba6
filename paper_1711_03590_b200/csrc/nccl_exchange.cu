// Native ghost exchange on the device. Replaces the reference GhostExchanger
// (ghost_exchange.cpp:300-398), whose transport is an in-process byte queue,
// with grouped point-to-point transfers on a dedicated communication stream:
//   start_update : pack owned interface cells (plan order; whole-cell plans
//                  as cell slot lists) and post the sends; receives land
//                  directly in u's ghost region (plan order == ghost storage
//                  order, verified at setup), partial plans via a buffer;
//   finish_update: the compute stream waits for the receives;
//   compress     : ghost contributions travel back along the reversed
//                  routes and are added into the owned cells one neighbour
//                  at a time in ascending rank order (deterministic), then
//                  y's ghost region is zeroed.
// Transports: NCCL send/recv (libnccl.so.2 opened at run time, so single-GPU
// use has no NCCL dependency and the process reuses torch's NCCL if it is
// already loaded), and an in-process loopback (R rank operators in one
// process, one cudaMemcpyAsync per message) that runs this exact exchanger
// -- packing, in-place receives, compress and accumulation order -- on one
// GPU.
#include "nccl_exchange.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
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

// hooks: C frames, so every exception becomes a status code + message
template <typename F>
dgx_status hook_guard(F &&f)
{
  try
    {
      f();
      return DGX_OK;
    }
  catch (const Error &e)
    {
      set_last_error(e.what());
      return static_cast<dgx_status>(e.code);
    }
  catch (const std::exception &e)
    {
      set_last_error(e.what());
      return DGX_RUNTIME_ERROR;
    }
  catch (...)
    {
      set_last_error("unknown error in an exchange hook");
      return DGX_RUNTIME_ERROR;
    }
}

dgx_status hook_start(void *ctx, void *v, void *s)
{
  return hook_guard([&] { static_cast<Exchanger *>(ctx)->start_update(v, static_cast<cudaStream_t>(s)); });
}
dgx_status hook_finish(void *ctx, void *v, void *s)
{
  return hook_guard([&] { static_cast<Exchanger *>(ctx)->finish_update(v, static_cast<cudaStream_t>(s)); });
}
dgx_status hook_compress(void *ctx, void *v, void *s)
{
  return hook_guard([&] { static_cast<Exchanger *>(ctx)->compress(v, static_cast<cudaStream_t>(s)); });
}

class NcclTransport final : public Transport
{
public:
  NcclTransport(const void *id128, int n_ranks, int rank)
  {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t comm;
    nccl_check(nccl().CommInitRank(&comm, n_ranks, id, rank), "ncclCommInitRank");
    comm_ = comm;
  }
  ~NcclTransport() override
  {
    if (comm_ && nccl().CommDestroy)
      nccl().CommDestroy(comm_);
  }
  void group_start() override { nccl_check(nccl().GroupStart(), "ncclGroupStart"); }
  void send(const void *buf, long long count, int elem, int peer, cudaStream_t s) override
  {
    nccl_check(nccl().Send(buf, count, elem == 4 ? ncclFloat : ncclDouble, peer, comm_, s), "ncclSend");
  }
  void recv(void *buf, long long count, int elem, int peer, cudaStream_t s) override
  {
    nccl_check(nccl().Recv(buf, count, elem == 4 ? ncclFloat : ncclDouble, peer, comm_, s), "ncclRecv");
  }
  void group_end(cudaStream_t) override { nccl_check(nccl().GroupEnd(), "ncclGroupEnd"); }

private:
  ncclComm_t comm_ = nullptr;
};
} // namespace

// ---- loopback transport ---------------------------------------------------

class LoopbackWorld
{
public:
  explicit LoopbackWorld(int n) : n_ranks(n) {}
  struct Msg
  {
    const void *src = nullptr;
    long long bytes = 0;
    cudaEvent_t ready = nullptr; // sender: packed
    cudaEvent_t done = nullptr;  // receiver: copied
    bool consumed = false;
  };
  const int n_ranks;
  std::mutex m;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box; // (src, dst) FIFO
};

namespace
{
class LoopbackTransport final : public Transport
{
public:
  LoopbackTransport(std::shared_ptr<LoopbackWorld> w, int rank) : w_(std::move(w)), rank_(rank)
  {
    if (rank < 0 || rank >= w_->n_ranks)
      fail(Code::invalid_argument, "loopback transport: rank out of range");
  }
  void group_start() override { pend_.clear(); }
  void send(const void *buf, long long count, int elem, int peer, cudaStream_t) override
  {
    pend_.push_back({true, const_cast<void *>(buf), count * elem, peer});
  }
  void recv(void *buf, long long count, int elem, int peer, cudaStream_t) override
  {
    pend_.push_back({false, buf, count * elem, peer});
  }
  void group_end(cudaStream_t s) override
  {
    using namespace std::chrono_literals;
    cudaEvent_t ready;
    cuda_check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(ready, s), "cudaEventRecord");
    std::vector<std::shared_ptr<LoopbackWorld::Msg>> mine;
    std::unique_lock<std::mutex> lk(w_->m);
    for (const Pending &p : pend_)
      if (p.send)
        {
          auto msg = std::make_shared<LoopbackWorld::Msg>();
          msg->src = p.buf;
          msg->bytes = p.bytes;
          msg->ready = ready;
          cuda_check(cudaEventCreateWithFlags(&msg->done, cudaEventDisableTiming), "cudaEventCreate");
          w_->box[{rank_, p.peer}].push_back(msg);
          mine.push_back(msg);
        }
    w_->cv.notify_all();
    for (const Pending &p : pend_)
      {
        if (p.send)
          continue;
        auto &q = w_->box[{p.peer, rank_}];
        if (!w_->cv.wait_for(lk, 120s, [&] { return !q.empty(); }))
          fail(Code::runtime_error, "loopback exchange: no message from rank " + std::to_string(p.peer) +
                                      " (timeout)");
        auto msg = q.front();
        q.pop_front();
        if (msg->bytes != p.bytes)
          fail(Code::runtime_error, "GhostExchanger: message size does not match the plan");
        cuda_check(cudaStreamWaitEvent(s, msg->ready, 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(p.buf, msg->src, p.bytes, cudaMemcpyDefault, s), "loopback copy");
        cuda_check(cudaEventRecord(msg->done, s), "cudaEventRecord");
        msg->consumed = true;
        w_->cv.notify_all();
      }
    for (auto &msg : mine)
      {
        if (!w_->cv.wait_for(lk, 120s, [&] { return msg->consumed; }))
          fail(Code::runtime_error, "loopback exchange: message never received (timeout)");
        // the sender may reuse its buffer only after the copy
        cuda_check(cudaStreamWaitEvent(s, msg->done, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(msg->done);
      }
    lk.unlock();
    cudaEventDestroy(ready); // every waiter captured it already
    pend_.clear();
  }

private:
  struct Pending
  {
    bool send;
    void *buf;
    long long bytes;
    int peer;
  };
  std::shared_ptr<LoopbackWorld> w_;
  int rank_;
  std::vector<Pending> pend_;
};

template <typename F>
void typed(int elem, F &&f)
{
  if (elem == 8)
    f(double{});
  else
    f(float{});
}
} // namespace

std::shared_ptr<LoopbackWorld> make_loopback_world(int n_ranks)
{
  if (n_ranks < 1)
    fail(Code::invalid_argument, "loopback world: n_ranks must be >= 1");
  return std::make_shared<LoopbackWorld>(n_ranks);
}

std::unique_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackWorld> w, int rank)
{
  return std::make_unique<LoopbackTransport>(std::move(w), rank);
}

std::unique_ptr<Transport> make_nccl_transport(const void *id128, int n_ranks, int rank)
{
  return std::make_unique<NcclTransport>(id128, n_ranks, rank);
}

void nccl_unique_id(void *id128)
{
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof id);
}

Exchanger *native_exchanger(const dgx_hooks *h)
{
  if (h && h->start_ghost_update == hook_start && h->finish_ghost_update == hook_finish &&
      h->compress == hook_compress && h->ctx)
    return static_cast<Exchanger *>(h->ctx);
  return nullptr;
}

Exchanger::Exchanger(Operator *op, std::unique_ptr<Transport> t) : op_(op), tr_(std::move(t))
{
  cuda_check(cudaSetDevice(op->device()), "cudaSetDevice");
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
  tr_.reset();
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

// update_ghost_values (ghost_exchange.cpp:300-351): pack the plan values,
// one grouped send/recv per neighbour on the exchange stream; whole ghost
// cells land in place in the ghost region, partial (Hermite 2-layer) plans
// through a buffer and an indexed unpack.
void Exchanger::start_update(void *u, cudaStream_t s)
{
  if (in_flight_)
    fail(Code::logic_error, "update_ghost_values: update already in flight");
  const RankLayout &l = op_->layout();
  const auto &so = op_->send_offsets(), &ro = op_->recv_offsets();
  cuda_check(cudaEventRecord(ev_ready_, s), "event record");
  cuda_check(cudaStreamWaitEvent(comm_stream_, ev_ready_, 0), "wait");
  typed(elem_, [&](auto t) {
    using T = decltype(t);
    if (op_->whole_cells())
      launch_gather_cells<T>(static_cast<const T *>(u), op_->send_slots().get(),
                             op_->send_cell_offsets().back(), (int)op_->nq(),
                             reinterpret_cast<T *>(send_buf_.get()), comm_stream_);
    else
      launch_gather_values<T>(static_cast<const T *>(u), op_->send_index().get(), so.back(),
                              reinterpret_cast<T *>(send_buf_.get()), comm_stream_);
  });
  char *ub = static_cast<char *>(u);
  char *sb = reinterpret_cast<char *>(send_buf_.get());
  char *rb = op_->recv_in_place() ? ub + l.owned_size() * elem_
                                  : reinterpret_cast<char *>(recv_buf_.get());
  tr_->group_start();
  for (std::size_t i = 0; i < l.send.size(); ++i)
    tr_->send(sb + so[i] * elem_, so[i + 1] - so[i], elem_, l.send[i].neighbor, comm_stream_);
  for (std::size_t i = 0; i < l.recv.size(); ++i)
    tr_->recv(rb + ro[i] * elem_, ro[i + 1] - ro[i], elem_, l.recv[i].neighbor, comm_stream_);
  tr_->group_end(comm_stream_);
  if (!op_->recv_in_place())
    typed(elem_, [&](auto t) {
      using T = decltype(t);
      launch_scatter_values<T>(static_cast<T *>(u), op_->recv_index().get(), ro.back(),
                               reinterpret_cast<const T *>(rb), comm_stream_);
    });
  cuda_check(cudaEventRecord(ev_done_, comm_stream_), "event record");
  in_flight_ = true;
}

void Exchanger::finish_update(void *, cudaStream_t s)
{
  if (!in_flight_)
    fail(Code::logic_error, "finish_ghost_update: no update was started on this vector");
  cuda_check(cudaStreamWaitEvent(s, ev_done_, 0), "wait");
  in_flight_ = false;
}

// compress (ghost_exchange.cpp:359-398): the ghost contributions travel the
// reversed update routes ...
void Exchanger::compress_post(void *y, cudaStream_t s_ghost)
{
  if (in_flight_)
    {
      cuda_check(cudaStreamWaitEvent(s_ghost, ev_done_, 0), "wait");
      in_flight_ = false;
    }
  const RankLayout &l = op_->layout();
  const auto &so = op_->send_offsets(), &ro = op_->recv_offsets();
  cuda_check(cudaEventRecord(ev_ready_, s_ghost), "event record");
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
  tr_->group_start();
  for (std::size_t i = 0; i < l.recv.size(); ++i)
    tr_->send(gb + ro[i] * elem_, ro[i + 1] - ro[i], elem_, l.recv[i].neighbor, comm_stream_);
  for (std::size_t i = 0; i < l.send.size(); ++i)
    tr_->recv(rb + so[i] * elem_, so[i + 1] - so[i], elem_, l.send[i].neighbor, comm_stream_);
  tr_->group_end(comm_stream_);
  cuda_check(cudaEventRecord(ev_done_, comm_stream_), "event record");
  compress_posted_ = true;
}

// ... and are added into the owned cells in ascending neighbour rank, then
// y's ghost region is zeroed
void Exchanger::compress_finish(void *y, cudaStream_t s)
{
  if (!compress_posted_)
    fail(Code::logic_error, "compress: nothing was posted");
  compress_posted_ = false;
  const RankLayout &l = op_->layout();
  const auto &so = op_->send_offsets();
  const auto &sco = op_->send_cell_offsets();
  char *yb = static_cast<char *>(y);
  const char *rb = reinterpret_cast<const char *>(recv_buf_.get());
  cuda_check(cudaStreamWaitEvent(s, ev_done_, 0), "wait");
  for (std::size_t i = 0; i < l.send.size(); ++i)
    typed(elem_, [&](auto t) {
      using T = decltype(t);
      const T *src = reinterpret_cast<const T *>(rb) + so[i];
      if (op_->whole_cells())
        launch_scatter_add_cells<T>(static_cast<T *>(y), op_->send_slots().get() + sco[i], sco[i + 1] - sco[i],
                                    (int)op_->nq(), src, s);
      else
        launch_scatter_add_values<T>(static_cast<T *>(y), op_->send_index().get() + so[i], so[i + 1] - so[i],
                                     src, s);
    });
  const long long ghost_vals = l.total_size() - l.owned_size();
  if (ghost_vals > 0)
    cuda_check(cudaMemsetAsync(yb + l.owned_size() * elem_, 0, ghost_vals * elem_, s), "memset");
}

void Exchanger::compress(void *y, cudaStream_t s)
{
  compress_post(y, s);
  compress_finish(y, s);
}

} // namespace dgx
