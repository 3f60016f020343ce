// step_zfp_b.cu -- zfp-mode step kernels for rates 17..32 (see step_launch.cuh).
#include "codec_zfp.cuh"
#include "step_launch.cuh"

namespace hccx {

cudaError_t launch_zfp_b(int rate, int op, const StepParams& p, cudaStream_t s) {
  switch (rate) {
    case 17: return launch_codec_step<ZfpRateCodec<17>>(op, p, s);
    case 18: return launch_codec_step<ZfpRateCodec<18>>(op, p, s);
    case 19: return launch_codec_step<ZfpRateCodec<19>>(op, p, s);
    case 20: return launch_codec_step<ZfpRateCodec<20>>(op, p, s);
    case 21: return launch_codec_step<ZfpRateCodec<21>>(op, p, s);
    case 22: return launch_codec_step<ZfpRateCodec<22>>(op, p, s);
    case 23: return launch_codec_step<ZfpRateCodec<23>>(op, p, s);
    case 24: return launch_codec_step<ZfpRateCodec<24>>(op, p, s);
    case 25: return launch_codec_step<ZfpRateCodec<25>>(op, p, s);
    case 26: return launch_codec_step<ZfpRateCodec<26>>(op, p, s);
    case 27: return launch_codec_step<ZfpRateCodec<27>>(op, p, s);
    case 28: return launch_codec_step<ZfpRateCodec<28>>(op, p, s);
    case 29: return launch_codec_step<ZfpRateCodec<29>>(op, p, s);
    case 30: return launch_codec_step<ZfpRateCodec<30>>(op, p, s);
    case 31: return launch_codec_step<ZfpRateCodec<31>>(op, p, s);
    case 32: return launch_codec_step<ZfpRateCodec<32>>(op, p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
