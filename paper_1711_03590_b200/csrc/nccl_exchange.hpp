#pragma once

#include "operator.hpp"

#include <memory>

namespace dgx
{

void nccl_unique_id(void *id128);

// Point-to-point transport under the exchanger: grouped sends / receives of
// byte ranges between rank-local device buffers, ordered on a stream (the
// role of the reference's in-process byte queues, ghost_exchange.cpp:409-430).
class Transport
{
public:
  virtual ~Transport() = default;
  virtual void group_start() = 0;
  virtual void send(const void *buf, long long count, int elem, int peer, cudaStream_t s) = 0;
  virtual void recv(void *buf, long long count, int elem, int peer, cudaStream_t s) = 0;
  // every send / receive of the group is ordered on s when this returns
  virtual void group_end(cudaStream_t s) = 0;
};

// NCCL send/recv (NVLink 5 / NVSwitch between the GPUs of one box)
std::unique_ptr<Transport> make_nccl_transport(const void *id128, int n_ranks, int rank);

// In-process loopback: R rank operators (one GPU or several) in one process,
// each rank's applies on its own host thread; a send is matched with the
// peer's receive and becomes one cudaMemcpyAsync between the two device
// buffers on the receiver's stream (the sender's stream waits for it).
class LoopbackWorld;
std::shared_ptr<LoopbackWorld> make_loopback_world(int n_ranks);
std::unique_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackWorld> w, int rank);

// GhostExchanger (ghost_exchange.hpp:96-128) on the device over a transport.
class Exchanger
{
public:
  Exchanger(Operator *op, std::unique_ptr<Transport> t);
  ~Exchanger();
  Exchanger(const Exchanger &) = delete;
  Exchanger &operator=(const Exchanger &) = delete;

  dgx_hooks hooks();
  void start_update(void *u, cudaStream_t s);
  void finish_update(void *u, cudaStream_t s);
  void compress(void *y, cudaStream_t s);
  // compress split in two: the ghost contributions leave once s_ghost (the
  // ghost-coupled phase) is done; the owner accumulates them on s
  void compress_post(void *y, cudaStream_t s_ghost);
  void compress_finish(void *y, cudaStream_t s);
  Operator *op() const { return op_; }

private:
  Operator *op_;
  std::unique_ptr<Transport> tr_;
  cudaStream_t comm_stream_ = nullptr;
  cudaEvent_t ev_ready_ = nullptr, ev_done_ = nullptr;
  DeviceArray<double> send_buf_, recv_buf_, ghost_buf_;
  int elem_ = 8;
  bool in_flight_ = false, compress_posted_ = false;
};

// the exchanger behind hooks returned by Exchanger::hooks(), else null
Exchanger *native_exchanger(const dgx_hooks *hooks);

// capi.cpp: keep a message for dgx_last_error() (hooks report errors as
// status codes: exceptions never cross their C frames)
void set_last_error(const char *msg);

} // namespace dgx
