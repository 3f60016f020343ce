// fused_fr_hi.cu -- NVLink engine kernels, fixed-rate 17..32 (see fused_launch.cuh).
#include "codec_fixed_rate.cuh"
#include "fused_launch.cuh"

namespace hccx {

cudaError_t launch_fused_fr_hi(int rate, const FusedParams* p, int nv, cudaStream_t s) {
  switch (rate) {
    case 17: return launch_fused_codec<FixedRateCodec<17>>(p, nv, s);
    case 18: return launch_fused_codec<FixedRateCodec<18>>(p, nv, s);
    case 19: return launch_fused_codec<FixedRateCodec<19>>(p, nv, s);
    case 20: return launch_fused_codec<FixedRateCodec<20>>(p, nv, s);
    case 21: return launch_fused_codec<FixedRateCodec<21>>(p, nv, s);
    case 22: return launch_fused_codec<FixedRateCodec<22>>(p, nv, s);
    case 23: return launch_fused_codec<FixedRateCodec<23>>(p, nv, s);
    case 24: return launch_fused_codec<FixedRateCodec<24>>(p, nv, s);
    case 25: return launch_fused_codec<FixedRateCodec<25>>(p, nv, s);
    case 26: return launch_fused_codec<FixedRateCodec<26>>(p, nv, s);
    case 27: return launch_fused_codec<FixedRateCodec<27>>(p, nv, s);
    case 28: return launch_fused_codec<FixedRateCodec<28>>(p, nv, s);
    case 29: return launch_fused_codec<FixedRateCodec<29>>(p, nv, s);
    case 30: return launch_fused_codec<FixedRateCodec<30>>(p, nv, s);
    case 31: return launch_fused_codec<FixedRateCodec<31>>(p, nv, s);
    case 32: return launch_fused_codec<FixedRateCodec<32>>(p, nv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
