// adamw_math.cuh — the per-element AdamW update ("AdamW"; reading R11),
// shared by the flat optimizer kernel (kernels.cu) and the weight-gradient GEMM epilogue
// that applies it in place of storing dW (gemm.cu, EPI_ADAMW), so that both produce the
// same fp32 arithmetic.
#pragma once

namespace slip {

// g: the summed gradient; m, v, p updated in place; wdl = weight decay of this element (0
// for biases / LayerNorm); inv_bc1 / inv_bc2 = 1 / (1 - beta^step).  Every operation is an
// explicitly rounded intrinsic (no FMA contraction left to the compiler), so the kernels
// that share this function produce bit-identical results:
//   m <- b1 m + (1 - b1) g',  v <- b2 v + (1 - b2) g'^2,  g' = grad_scale g
//   p <- p - lr wd p - lr (m / bc1) / (sqrt(v / bc2) + eps)
__device__ __forceinline__ void adamw_update(float& p, float& m, float& v, float g, float lr, float b1, float b2,
                                             float eps, float wdl, float inv_bc1, float inv_bc2, float grad_scale) {
  const float gr = __fmul_rn(grad_scale, g);
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(__fsub_rn(1.f, b1), gr));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fmul_rn(__fsub_rn(1.f, b2), gr), gr));
  const float mh = __fmul_rn(m, inv_bc1);
  const float vh = __fmul_rn(v, inv_bc2);
  const float upd = __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps));
  p = __fsub_rn(__fsub_rn(p, __fmul_rn(__fmul_rn(lr, wdl), p)), upd);
}

}  // namespace slip
