// jf_comm.cu — stand-alone use of the in-kernel cross-rank combine
// (jf_pass.cuh comm_combine): the startup all-reduce of the global point
// count m (jf.h jf_opts.m_global = 0; reading R6 needs the global m) and the
// combine-latency probe behind jf_comm_bench.
#include "jf_pass.cuh"

namespace jf {

__global__ void comm_sum_kernel(CommDev cd, unsigned long long epoch, double v, double* out, int* err) {
  __shared__ double vec[KMAX];
  for (int k = threadIdx.x; k < KMAX; k += blockDim.x) vec[k] = (k == 0) ? v : 0.0;
  __syncthreads();
  const bool ok = comm_combine<KMAX, 32>(cd, epoch, vec);
  if (threadIdx.x == 0) {
    *out = vec[0];
    *err = ok ? 0 : -5;
  }
}

// One combine (v in slot 0 of a KMAX-double vector) across the ranks of cd,
// epoch-numbered like the pass kernels' combines.
int launch_comm_sum(const CommDev& cd, unsigned long long epoch, double v, double* d_out, int* d_err, cudaStream_t s) {
  comm_sum_kernel<<<1, 32, 0, s>>>(cd, epoch, v, d_out, d_err);
  return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

const void* comm_sum_kernel_ptr() { return (const void*)comm_sum_kernel; }

}  // namespace jf
