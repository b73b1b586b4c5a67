// Single-call secure / plain bilinear layers over the C ABI (SURVEY.md §8(b)
// minimum exports): each composes the engine's own launches — operand limb
// packs, the tcgen05 ring GEMM and the fused reshare + truncate epilogue —
// into ONE extern "C" call with a caller-provided workspace, so a binding
// (ctypes / cgo / JNI) replaces the reference's
//   ring.bilinear_exact(x, w, conv2d_spec(...))          ring.py:183-256
//   protocols.matmul_shares(ctx, x, y, bits)             protocols.py:97-117
//   protocols.conv2d_shares(ctx, x, k, stride, pad, bits) protocols.py:120-136
// with one function each.  Trio tensors are contiguous (3, ...) u64 buffers
// (component c_i in plane i; party i holds (c_i, c_{i+1})).  The PRF
// counters (ARITH_ZERO, TRUNC_RHO, TRUNC_R) are the ones the host allotted by
// mirroring the reference's lockstep `take` (sharing.py:225-230).
#include <cuda_runtime.h>
#include <string.h>

#include "common.cuh"
#include "launch.cuh"

namespace {

constexpr int64_t kAlign = 256;
constexpr int64_t kMaxAcc = 1 << 20;  // ring.py:191-195 accumulation bound

int64_t up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct ConvGeom {
  int64_t n, c, h, w, o, kh, kw, sh, sw, ph, pw, oh, ow, M, K;
  bool ok;
};

ConvGeom conv_geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw, int sh, int sw, int ph,
                   int pw) {
  ConvGeom g{N, C, H, W, O, kh, kw, sh, sw, ph, pw, 0, 0, 0, 0, false};
  if (N < 0 || C < 1 || O < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0) return g;
  if (H + 2 * ph < kh || W + 2 * pw < kw) return g;
  g.oh = (H + 2 * ph - kh) / sh + 1;
  g.ow = (W + 2 * pw - kw) / sw + 1;
  g.M = N * g.oh * g.ow;
  g.K = C * kh * kw;
  g.ok = true;
  return g;
}

mpc3_operand im2col_operand(const ConvGeom& g) {
  mpc3_operand o;
  memset(&o, 0, sizeof(o));
  o.mode = MPC3_GATHER_IM2COL;
  o.rows = g.M;
  o.k = g.K;
  o.n = g.n;
  o.c = g.c;
  o.h = g.h;
  o.w = g.w;
  o.sN = g.c * g.h * g.w;
  o.sC = g.h * g.w;
  o.sH = g.w;
  o.sW = 1;
  o.kh = g.kh;
  o.kw = g.kw;
  o.sh = g.sh;
  o.sw = g.sw;
  o.ph = g.ph;
  o.pw = g.pw;
  o.dh = 1;
  o.dw = 1;
  o.oh = g.oh;
  o.ow = g.ow;
  return o;
}

// rows x k, element (r, k) at off + r * s_r + k * t2 (a plain 2-d view)
mpc3_operand dense_operand(int64_t rows, int64_t k, int64_t s_r, int64_t t2) {
  mpc3_operand o;
  memset(&o, 0, sizeof(o));
  o.mode = MPC3_GATHER_DENSE;
  o.rows = rows;
  o.k = k;
  o.s_r = s_r;
  o.t2 = t2;
  o.K1 = 1;
  o.K2 = k;
  return o;
}

mpc3_view4 view4(int64_t n0, int64_t n1, int64_t n2, int64_t n3, const int64_t zs[4]) {
  mpc3_view4 v;
  const int64_t full[4] = {n0, n1, n2, n3};
  for (int i = 0; i < 4; ++i) {
    v.full[i] = full[i];
    v.origin[i] = 0;
    v.crop[i] = full[i];
    v.z_stride[i] = zs[i];
  }
  v.out_stride[3] = 1;
  v.out_stride[2] = n3;
  v.out_stride[1] = n3 * n2;
  v.out_stride[0] = n3 * n2 * n1;
  v.z_plane = v.out_plane = n0 * n1 * n2 * n3;
  return v;
}

// Workspace of a secure bilinear layer: A = the left operand once per
// component (role 3), B = the right operand's cross-term halves (role 0,
// halves at the 32-aligned kc), z = the three parties' cross terms.
struct SecureWs {
  int64_t kpa, kc, a_bytes, b_bytes, z_bytes;
};
SecureWs secure_ws(int64_t M, int64_t N, int64_t K) {
  SecureWs s;
  s.kpa = up(K, 32);
  s.kc = up(K, 32);
  s.a_bytes = up(3 * 8 * M * s.kpa, kAlign);
  s.b_bytes = up(3 * 8 * N * 2 * s.kc, kAlign);
  s.z_bytes = up(3 * M * N * 8, kAlign);
  return s;
}

// z_i = (x_i + x_{i+1}) y_i + x_i y_{i+1} for the three parties (protocols.py:110-115)
// as one batched ring GEMM, then reshare + truncate through `view`.
int secure_layer(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r, int bits,
                 const uint64_t* a_src, int64_t a_plane, const mpc3_operand& a_op, const uint64_t* b_src,
                 int64_t b_plane, const mpc3_operand& b_op, int64_t M, int64_t N, int64_t K, int c_col,
                 const mpc3_view4& view, uint64_t* out, void* workspace, void* stream) {
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;  // protocols.py:185-186
  if (K > kMaxAcc) return MPC3_ERR_EXACTNESS;
  if (!workspace || !out || !a_src || !b_src) return MPC3_ERR_CONFIG;
  const SecureWs s = secure_ws(M, N, K);
  uint8_t* A = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* B = A + s.a_bytes;
  uint64_t* z = reinterpret_cast<uint64_t*>(B + s.b_bytes);
  const int zeroed = mpc3_ring_gemm_needs_zero(1, 3, M, N, 2 * s.kc) == 1;
  int st = mpc3_ring_pack_halves(b_src, b_plane, &b_op, 0, B, 2 * s.kc, s.kc, stream);
  if (st) return st;
  st = mpc3_ring_pack_halves_z(a_src, a_plane, &a_op, 3, A, s.kpa, K, zeroed ? z : nullptr, zeroed ? 3 * M * N : 0,
                               stream);
  if (st) return st;
  st = mpc3_ring_gemm_t_z(A, 2, M, s.kpa, 0, B, 0, N, 2 * s.kc, 0, z, 3, M, N, s.kc, c_col, zeroed, stream);
  if (st) return st;
  return mpc3_rss_reshare_truncate(rk3, ctr, j_arith, j_rho, j_r, bits, z, &view, out, 0, stream);
}

__global__ void col_to_nchw_kernel(const uint64_t* __restrict__ z, uint64_t* __restrict__ y, int64_t N, int64_t O,
                                   int64_t P) {
  const int64_t n_out = N * O * P;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_out; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = f % P, o = (f / P) % O, n = f / (O * P);
    y[f] = z[o * (N * P) + n * P + p];  // column-major GEMM output (m = (n, p), o) -> NCHW
  }
}

}  // namespace

extern "C" {

size_t mpc3_ring_conv2d_workspace(int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw, int sh,
                                  int sw, int ph, int pw) {
  const ConvGeom g = conv_geom(N, C, H, W, O, kh, kw, sh, sw, ph, pw);
  if (!g.ok) return 0;
  const int64_t kp = up(g.K, 32);
  return (size_t)(up(8 * g.M * kp, kAlign) + up(8 * O * kp, kAlign) + up(8 * g.M * O, kAlign));
}

int mpc3_ring_conv2d_u64(const uint64_t* x, const uint64_t* w, uint64_t* y, int64_t N, int64_t C, int64_t H,
                         int64_t W, int64_t O, int kh, int kw, int sh, int sw, int ph, int pw, void* workspace,
                         void* stream) {
  const ConvGeom g = conv_geom(N, C, H, W, O, kh, kw, sh, sw, ph, pw);
  if (!g.ok) return MPC3_ERR_SHAPE;
  if (g.K > kMaxAcc) return MPC3_ERR_EXACTNESS;
  if (g.M == 0) return MPC3_OK;
  if (!x || !w || !y || !workspace) return MPC3_ERR_CONFIG;
  const int64_t kp = up(g.K, 32);
  uint8_t* A = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* B = A + up(8 * g.M * kp, kAlign);
  uint64_t* z = reinterpret_cast<uint64_t*>(B + up(8 * O * kp, kAlign));
  const mpc3_operand oa = im2col_operand(g);
  const mpc3_operand ob = dense_operand(O, g.K, g.K, 1);
  int st = mpc3_ring_pack(x, 0, &oa, 2, A, kp, stream);
  if (st) return st;
  st = mpc3_ring_pack(w, 0, &ob, 2, B, kp, stream);
  if (st) return st;
  st = mpc3_ring_gemm_auto(A, B, z, 1, g.M, O, kp, 1, stream);
  if (st) return st;
  const int64_t n = g.M * O;
  col_to_nchw_kernel<<<mpc3::grid_for((uint64_t)n, 256), 256, 0, (cudaStream_t)stream>>>(z, y, N, O, g.oh * g.ow);
  return cudaGetLastError() == cudaSuccess ? MPC3_OK : MPC3_ERR_CUDA;
}

size_t mpc3_rss_matmul_workspace(int64_t M, int64_t K, int64_t N) {
  const SecureWs s = secure_ws(M, N, K);
  return (size_t)(s.a_bytes + s.b_bytes + s.z_bytes);
}

int mpc3_rss_matmul_reshare_trunc(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                  uint64_t j_r, int bits, const uint64_t* x, const uint64_t* y, uint64_t* out,
                                  int64_t M, int64_t K, int64_t N, void* workspace, void* stream) {
  if (M < 0 || K < 1 || N < 1) return MPC3_ERR_SHAPE;
  if (M == 0) return MPC3_OK;
  const mpc3_operand a = dense_operand(M, K, K, 1);  // x (M, K) row-major per component
  const mpc3_operand b = dense_operand(N, K, 1, N);  // y (K, N): row n of B^T = column n of y
  const int64_t zs[4] = {0, 0, N, 1};                // z row-major (M, N) per party
  const mpc3_view4 v = view4(1, 1, M, N, zs);
  return secure_layer(rk3, ctr, j_arith, j_rho, j_r, bits, x, M * K, a, y, K * N, b, M, N, K, 0, v, out, workspace,
                      stream);
}

size_t mpc3_rss_conv2d_workspace(int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw, int sh,
                                 int sw, int ph, int pw) {
  const ConvGeom g = conv_geom(N, C, H, W, O, kh, kw, sh, sw, ph, pw);
  if (!g.ok) return 0;
  const SecureWs s = secure_ws(g.M, O, g.K);
  return (size_t)(s.a_bytes + s.b_bytes + s.z_bytes);
}

int mpc3_rss_conv2d_reshare_trunc(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                  uint64_t j_r, int bits, const uint64_t* x, const uint64_t* w, uint64_t* out,
                                  int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw, int sh,
                                  int sw, int ph, int pw, void* workspace, void* stream) {
  const ConvGeom g = conv_geom(N, C, H, W, O, kh, kw, sh, sw, ph, pw);
  if (!g.ok) return MPC3_ERR_SHAPE;
  if (g.M == 0) return MPC3_OK;
  const mpc3_operand a = im2col_operand(g);
  const mpc3_operand b = dense_operand(O, g.K, g.K, 1);  // w (O, C, kh, kw): row o, K contiguous
  // z[(n, y, x), o] column-major: each (n, o) plane's (y, x) run contiguous
  const int64_t zs[4] = {g.oh * g.ow, g.M, g.ow, 1};
  const mpc3_view4 v = view4(N, O, g.oh, g.ow, zs);
  return secure_layer(rk3, ctr, j_arith, j_rho, j_r, bits, x, N * C * H * W, a, w, O * g.K, b, g.M, O, g.K, 1, v, out,
                      workspace, stream);
}

}  // extern "C"
