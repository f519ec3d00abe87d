// Internal: the communicator behind fp8_comm_t (NCCL, one rank per GPU).
#pragma once
#include <nccl.h>

struct fp8_comm_s {
  ncclComm_t nccl;
  int nranks, rank;
};
