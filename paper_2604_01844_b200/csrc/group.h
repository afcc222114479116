// Internal interface of the multi-GPU group (group.cu). Error-returning functions give an
// empty string on success and the message otherwise (api.cu turns it into GSCT_ERR_CUDA).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/gsct_cuda.h"

namespace gsct_dev {

std::string group_new_id(unsigned char out[128]);
std::string group_create(int device, const unsigned char id[128], int n_ranks, int rank, gsct_group* out);
void group_destroy(gsct_group g);
int group_rank(gsct_group g);
int group_size(gsct_group g);
int group_device(gsct_group g);
std::string group_allreduce_sum_f64(gsct_group g, double* buf, size_t count, cudaStream_t st);
std::string group_allreduce_max_u8(gsct_group g, uint8_t* buf, size_t count, cudaStream_t st);
// every rank k broadcasts buf[offsets[k], offsets[k+1]) into the same range on all ranks
std::string group_allgather_slabs_f32(gsct_group g, float* buf, const size_t* offsets, cudaStream_t st);
int nccl_version();

}  // namespace gsct_dev
