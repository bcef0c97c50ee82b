// fio_comm.h -- NCCL plumbing of the wedge-sharded apply (fio_comm.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>

#include "../../include/fio.h"

namespace fio {

fio_status comm_unique_id(void* id_out /* FIO_NCCL_ID_BYTES */);
// ncclCommInitRank on the current device (collective over the nranks processes)
fio_status comm_create(const void* id_bytes, int nranks, int rank, void** comm_out);
void comm_destroy(void* comm);
// sum over ranks of `part` (nranks * slab_reals reals), rank r keeps reals [r slab_reals, (r+1) slab_reals)
fio_status comm_reduce_scatter(void* comm, const void* part, void* slab, size_t slab_reals, bool c64,
                               cudaStream_t s);
// in-place all-gather: rank r's slab_reals reals at full + r slab_reals are copied to every rank
fio_status comm_all_gather(void* comm, void* full, int rank, size_t slab_reals, bool c64, cudaStream_t s);

}  // namespace fio
