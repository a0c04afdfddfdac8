// nccl_put.hpp -- direct-put channel over NCCL symmetric windows (the NCCL
// 2.28 device API): peers' receive windows are reached by NVLink loads /
// stores through LSA pointers, and an LSA barrier kernel orders the stores
// before the combine (nccl_put.cu).
#pragma once

#include <memory>
#include <vector>

#include <nccl.h>

#include "transport.hpp"

namespace tetmf {

// collective over the communicator (window registration, device
// communicator, count all-gather); throws CommError when a peer is not
// load/store reachable (not in the LSA team) or NCCL fails
std::unique_ptr<PutChannel> nccl_open_put(ncclComm_t comm, int rank, int nranks, const std::vector<int>& peers,
                                          const std::vector<i64>& send_off, const std::vector<i64>& recv_off);

} // namespace tetmf
