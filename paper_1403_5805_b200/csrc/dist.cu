// dist.cu — row-block distribution over P GPUs, one process per GPU (§3.1).
//
// Rank r owns rows [r*m, (r+1)*m), m = n/P (P must divide n).  It holds its A rows,
// b and diag slices and two full-length x buffers.  Each sweep is followed, inside the same CUDA
// graph, by an in-place ncclAllGather of the new x slice (the MPI_Allgather scheme of PAPER.md:76,
// which the paper rejected for 100 Mbps Ethernet; NVSwitch makes every peer one hop away) and a
// one-scalar ncclAllReduce(max) of the bit pattern of max|dx| (replacing the MPI_Gather to rank 0
// of PAPER.md:96), so every rank takes the same stop decision.
#include "internal.h"
#include <cstring>

extern "C" int jacobi_partition(int64_t n, int nranks, int rank, int64_t* row0, int64_t* rows) {
  if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !rows)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_partition: bad argument");
  if (n % nranks != 0)
    return jacobi_set_error(JACOBI_EINDIVISIBLE, "nranks = " + std::to_string(nranks) + " does not divide n = " +
                                                     std::to_string(n) + " (PAPER.md:72 assumes p | n)");
  *rows = n / nranks;
  *row0 = (int64_t)rank * (n / nranks);
  return 0;
}

extern "C" int jacobi_nccl_unique_id(void* out128) {
  if (!out128) return jacobi_set_error(JACOBI_EINVAL, "jacobi_nccl_unique_id: NULL");
  ncclUniqueId id;
  JNCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

static int dist_create(jacobi_plan** out, const void* uid128, int rank, int nranks, int64_t n, int dtype,
                       const void* A_block, int64_t lda, int a_on_device, void* cuda_stream, bool colwise) {
  const char* fn = colwise ? "jacobi_dist_plan_create_colwise" : "jacobi_dist_plan_create";
  if (!out || !uid128 || !A_block || n < 1 || nranks < 1 || rank < 0 || rank >= nranks ||
      (dtype != JACOBI_F64 && dtype != JACOBI_F32))
    return jacobi_set_error(JACOBI_EINVAL, std::string(fn) + ": bad argument");
  int64_t row0 = 0, m = 0;
  int rc = jacobi_partition(n, nranks, rank, &row0, &m);
  if (rc) return rc;
  if (lda < (colwise ? m : n)) return jacobi_set_error(JACOBI_EINVAL, std::string(fn) + ": lda too small");
  if (colwise && nranks > 1 && m % 8 != 0)
    return jacobi_set_error(JACOBI_EINVAL, std::string(fn) + ": n / nranks must be a multiple of 8 (slab alignment)");
  jacobi_plan* p = new jacobi_plan();
  p->rank = rank;
  p->nranks = nranks;
  p->colwise = colwise;
  rc = colwise ? plan_init_common(p, n, m, row0, dtype, A_block, n, m, lda, a_on_device, cuda_stream)
               : plan_init_common(p, n, m, row0, dtype, A_block, m, n, lda, a_on_device, cuda_stream);
  if (rc == 0 && colwise) {
    cudaError_t e = cudaMalloc(&p->rsum, (size_t)n * 8);
    if (e == cudaSuccess) e = cudaMalloc(&p->rs_own, (size_t)m * 8);
    if (e != cudaSuccess) rc = jacobi_set_error(JACOBI_ENOMEM, std::string("column-wise buffers: ") + cudaGetErrorString(e));
  }
  if (rc == 0) {
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&p->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      p->comm = nullptr;
      rc = jacobi_set_error(JACOBI_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
  }
  unsigned long long zr = ~0ull;
  int nf = 0;
  if (rc == 0) rc = plan_validate_A(p, &zr, &nf);  // min-allreduce of the first zero row, max of the flag
  if (rc == 0 && zr != ~0ull)
    rc = jacobi_set_error(JACOBI_EZERODIAG, "a_ii == 0 at i = " + std::to_string(zr) + " (PAPER.md:53)");
  if (rc == 0 && nf) rc = jacobi_set_error(JACOBI_ENONFINITE, "A contains NaN or Inf");
  if (rc != 0) {
    std::string keep = jacobi_last_error();
    jacobi_plan_destroy(p);
    jacobi_set_error(rc, keep);
    return rc;
  }
  *out = p;
  return 0;
}

extern "C" int jacobi_dist_plan_create(jacobi_plan** out, const void* uid128, int rank, int nranks, int64_t n,
                                       int dtype, const void* A_rows, int64_t lda, int a_on_device,
                                       void* cuda_stream) {
  return dist_create(out, uid128, rank, nranks, n, dtype, A_rows, lda, a_on_device, cuda_stream, false);
}

extern "C" int jacobi_dist_plan_create_colwise(jacobi_plan** out, const void* uid128, int rank, int nranks,
                                               int64_t n, int dtype, const void* A_cols, int64_t lda,
                                               int a_on_device, void* cuda_stream) {
  return dist_create(out, uid128, rank, nranks, n, dtype, A_cols, lda, a_on_device, cuda_stream, true);
}
