// K10: the C4 operator, a 7-point Dirichlet Laplacian on an nx*ny*nz grid
// (x fastest), applied to an n x ncols block (krylov.py:129-130 ->
// operators.py:72-73).  Each output row accumulates its CSR row in
// ascending column order -- z-1, y-1, x-1, diagonal 6, x+1, y+1, z+1 --
// starting from 0, the order scipy's csr_matvecs uses on the Kronecker-sum
// matrix (bench.py:219-228 in 3-D), so results match the reference CSR
// operator bit for bit.  z-slab sharding: halo planes supply the z
// neighbours of the first / last local plane (NULL = Dirichlet boundary).
#include "common.cuh"

namespace rb {
namespace {

template <typename TX, typename TY>
__global__ void stencil7_kernel(int nx, int ny, int nzl, int ncols, const TX* __restrict__ X, int64_t ldx,
                                const TX* __restrict__ hlo, const TX* __restrict__ hhi, int64_t ldh,
                                TY* __restrict__ Y, int64_t ldy) {
  const int64_t plane = (int64_t)nx * ny;
  const int64_t n = plane * nzl;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= n || c >= ncols) return;
  const int x = (int)(r % nx);
  const int y = (int)((r / nx) % ny);
  const int z = (int)(r / plane);
  const TX* xc = X + (int64_t)c * ldx;
  double acc = 0.0;
  if (z > 0) acc += -(double)xc[r - plane];
  else if (hlo) acc += -(double)hlo[(r % plane) + (int64_t)c * ldh];
  if (y > 0) acc += -(double)xc[r - nx];
  if (x > 0) acc += -(double)xc[r - 1];
  acc = __dadd_rn(acc, __dmul_rn(6.0, (double)xc[r]));  // no FMA: scipy's loop rounds the product
  if (x < nx - 1) acc += -(double)xc[r + 1];
  if (y < ny - 1) acc += -(double)xc[r + nx];
  if (z < nzl - 1) acc += -(double)xc[r + plane];
  else if (hhi) acc += -(double)hhi[(r % plane) + (int64_t)c * ldh];
  Y[r + (int64_t)c * ldy] = (TY)acc;
}

}  // namespace

int stencil7(int xd, int yd, int nx, int ny, int nzl, int ncols, const void* X, int64_t ldx, const void* hlo,
             const void* hhi, int64_t ldh, void* Y, int64_t ldy, cudaStream_t st) {
  const int64_t n = (int64_t)nx * ny * nzl;
  RB_REQUIRE(nx >= 1 && ny >= 1 && nzl >= 1 && ncols >= 1 && ncols <= 65535 && X && Y && ldx >= n && ldy >= n,
             "rb_stencil7: bad args");
  RB_REQUIRE((!hlo && !hhi) || ldh >= (int64_t)nx * ny, "rb_stencil7: bad halo ld");
  dim3 grid(ceil_div(n, 256), ncols);
  if (xd == RB_F32 && yd == RB_F32)
    RB_KLAUNCH stencil7_kernel<float, float><<<grid, 256, 0, st>>>(nx, ny, nzl, ncols, (const float*)X, ldx, (const float*)hlo,
                                                        (const float*)hhi, ldh, (float*)Y, ldy);
  else if (xd == RB_F32)
    RB_KLAUNCH stencil7_kernel<float, double><<<grid, 256, 0, st>>>(nx, ny, nzl, ncols, (const float*)X, ldx, (const float*)hlo,
                                                         (const float*)hhi, ldh, (double*)Y, ldy);
  else if (yd == RB_F32)
    RB_KLAUNCH stencil7_kernel<double, float><<<grid, 256, 0, st>>>(nx, ny, nzl, ncols, (const double*)X, ldx,
                                                         (const double*)hlo, (const double*)hhi, ldh, (float*)Y, ldy);
  else
    RB_KLAUNCH stencil7_kernel<double, double><<<grid, 256, 0, st>>>(nx, ny, nzl, ncols, (const double*)X, ldx,
                                                          (const double*)hlo, (const double*)hhi, ldh, (double*)Y, ldy);
  return check_launch("rb_stencil7");
}

}  // namespace rb

namespace rb {
namespace {

template <typename TX, typename TY>
__global__ void csr_spmm_kernel(int64_t n, int ncols, const int64_t* __restrict__ indptr,
                                const int64_t* __restrict__ indices, const double* __restrict__ vals,
                                const TX* __restrict__ X, int64_t ldx, TY* __restrict__ Y, int64_t ldy) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= n || c >= ncols) return;
  const TX* xc = X + (int64_t)c * ldx;
  double acc = 0.0;
  for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(vals[e], (double)xc[indices[e]]));
  Y[r + (int64_t)c * ldy] = (TY)acc;
}

}  // namespace

int csr_spmm(int xd, int yd, int64_t n, int ncols, const int64_t* indptr, const int64_t* indices,
             const double* vals, const void* X, int64_t ldx, void* Y, int64_t ldy, cudaStream_t st) {
  RB_REQUIRE(n >= 0 && ncols >= 1 && ncols <= 65535 && indptr && X && Y && ldx >= n && ldy >= n,
             "rb_csr_spmm: bad args");
  if (n == 0) return RB_OK;
  dim3 grid(ceil_div(n, 256), ncols);
  if (xd == RB_F32 && yd == RB_F64)
    RB_KLAUNCH csr_spmm_kernel<float, double><<<grid, 256, 0, st>>>(n, ncols, indptr, indices, vals, (const float*)X, ldx,
                                                         (double*)Y, ldy);
  else if (xd == RB_F32)
    RB_KLAUNCH csr_spmm_kernel<float, float><<<grid, 256, 0, st>>>(n, ncols, indptr, indices, vals, (const float*)X, ldx,
                                                        (float*)Y, ldy);
  else if (yd == RB_F32)
    RB_KLAUNCH csr_spmm_kernel<double, float><<<grid, 256, 0, st>>>(n, ncols, indptr, indices, vals, (const double*)X, ldx,
                                                         (float*)Y, ldy);
  else
    RB_KLAUNCH csr_spmm_kernel<double, double><<<grid, 256, 0, st>>>(n, ncols, indptr, indices, vals, (const double*)X, ldx,
                                                          (double*)Y, ldy);
  return check_launch("rb_csr_spmm");
}

}  // namespace rb
