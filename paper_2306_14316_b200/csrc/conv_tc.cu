// tcgen05/TMEM tensor-core im2win convolution (TF32 / BF16 operands, fp32 accumulate).
// Placeholder until the kernel lands; the entry point fails loudly.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

size_t im2win_tc_workspace_bytes(int64_t c_out, int64_t K, int variant) {
  (void)variant;
  return static_cast<size_t>((K + 64) * (c_out + 256)) * 4 + 256;
}

int im2win_launch_conv_tc(const float*, const float*, float*, void*, int64_t, int64_t, int64_t, int64_t,
                          int64_t, int64_t, int, int, int, int, int, cudaStream_t, const char** err) {
  *err = "im2win_conv_f32: tensor-core variants are not built yet";
  return 3;
}
