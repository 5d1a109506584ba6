#pragma once

#include "operator.hpp"

namespace dgx
{

void nccl_unique_id(void *id128);

class Exchanger
{
public:
  Exchanger(Operator *op, const void *id128, int n_ranks);
  ~Exchanger();
  Exchanger(const Exchanger &) = delete;
  Exchanger &operator=(const Exchanger &) = delete;

  dgx_hooks hooks();
  dgx_status start_update(void *u, cudaStream_t s);
  dgx_status finish_update(void *u, cudaStream_t s);
  dgx_status compress(void *y, cudaStream_t s);

private:
  Operator *op_;
  void *comm_ = nullptr;
  cudaStream_t comm_stream_ = nullptr;
  cudaEvent_t ev_ready_ = nullptr, ev_done_ = nullptr;
  DeviceArray<double> send_buf_, recv_buf_, ghost_buf_;
  int elem_ = 8;
  bool in_flight_ = false;
};

} // namespace dgx
