// Debug harness: run fast_block vs exact_block on random bf16 blocks and report
// how often the fast path falls back, and any disagreement.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>
#include "../paper_2512_02010_b200/csrc/f46_device.cuh"
using namespace f46;

struct RegLoad { const float* x; __device__ float operator()(int i) const { return x[i]; } };

__global__ void k(const float* xs, int nblk, double alpha, int* stats, float* dbg) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const float* xb = xs + b * 16;
  float2 x[8]; float bmax = 0;
  for (int p = 0; p < 8; ++p) { x[p] = make_float2(xb[2*p], xb[2*p+1]); bmax = fmaxf(bmax, fmaxf(fabsf(x[p].x), fabsf(x[p].y))); }
  TensorConsts tc = make_consts(alpha, 0, DT_BF16);
  RegLoad ld{xb};
  BlockOut o, e;
  bool ok = fast_block<ADAPTIVE>(x, bmax, tc, ld, o);
  double xd[16]; for (int i = 0; i < 16; ++i) xd[i] = xb[i];
  exact_block(xd, alpha, ADAPTIVE, 0, &e);
  atomicAdd(&stats[0], ok ? 1 : 0);
  if (ok && (o.codes != e.codes || o.sc != e.sc || o.pick4 != e.pick4)) atomicAdd(&stats[1], 1);
  if (b < 8) {
    // recompute internals for printing
    const float alphaf = tc.alpha;
    uint32_t sc6 = block_scale_code(bmax, alphaf, 6.f, tc.r6_lo, tc.r6_hi), sc4 = block_scale_code(bmax, alphaf, 4.f, tc.r4_lo, tc.r4_hi);
    float d6 = e4m3_to_f32(sc6), d4 = e4m3_to_f32(sc4);
    Cand c6, c4; cand_eval(x, alphaf*d6, c6); cand_eval(x, alphaf*d4, c4);
    float D6 = alphaf*d6, D4 = alphaf*d4;
    float s6 = c6.sq*(D6*D6), s4 = c4.sq*(D4*D4);
    float tol = 0x1p-16f * bmax * (sqrt_approx(s6) + sqrt_approx(s4)) + 0x1p-14f * (s6 + s4) + 0x1p-32f * (bmax * bmax) + 0x1p-140f;
    dbg[b*8+0]=bmax; dbg[b*8+1]=d6; dbg[b*8+2]=d4; dbg[b*8+3]=c6.sq; dbg[b*8+4]=c4.sq; dbg[b*8+5]=s6; dbg[b*8+6]=s4; dbg[b*8+7]=tol;
  }
}

int main() {
  int nblk = 1 << 16;
  std::vector<float> h(nblk * 16);
  srand(1);
  float amax = 0;
  for (auto& v : h) {
    float u1 = (rand() + 1.f) / (RAND_MAX + 2.f), u2 = (rand() + 1.f) / (RAND_MAX + 2.f);
    float g = sqrtf(-2 * logf(u1)) * cosf(6.2831853f * u2);
    uint32_t b; memcpy(&b, &g, 4); b &= 0xFFFF0000u; memcpy(&g, &b, 4);  // bf16-representable
    v = g; amax = fmaxf(amax, fabsf(g));
  }
  double alpha = (double)(amax / 1536.0f);
  float *dx, *ddbg; int* ds;
  cudaMalloc(&dx, h.size() * 4); cudaMalloc(&ds, 8); cudaMalloc(&ddbg, 64 * 4);
  cudaMemcpy(dx, h.data(), h.size() * 4, cudaMemcpyHostToDevice); cudaMemset(ds, 0, 8);
  k<<<nblk / 128, 128>>>(dx, nblk, alpha, ds, ddbg);
  int st[2]; float dbg[64];
  cudaMemcpy(st, ds, 8, cudaMemcpyDeviceToHost); cudaMemcpy(dbg, ddbg, 256, cudaMemcpyDeviceToHost);
  printf("err=%s  blocks %d fast-ok %d (%.4f)  disagreements %d\n", cudaGetErrorString(cudaGetLastError()), nblk, st[0], st[0] / (double)nblk, st[1]);
  for (int b = 0; b < 8; ++b) printf("bmax %g d6 %g d4 %g sq6 %g sq4 %g s6 %g s4 %g tol %g\n", dbg[b*8], dbg[b*8+1], dbg[b*8+2], dbg[b*8+3], dbg[b*8+4], dbg[b*8+5], dbg[b*8+6], dbg[b*8+7]);
  return 0;
}
