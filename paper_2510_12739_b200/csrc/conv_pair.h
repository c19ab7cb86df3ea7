// conv_pair.h — launch interface of the CTA-pair (tcgen05 cta_group::2) 96 -> 96 channel 3x3
// convolution (conv_pair.cu).  Uses the same TcLaunch / TcGroup descriptors and weight image as
// conv_tc.cu's <96,96,3> kernel.
#pragma once
#include "conv_tc.h"

namespace cnrx {

// TcLaunch::flags bit: this launch uses the TMA-staged epilogue (residual load + output stores by TMA;
// set by the host when the staged shared-memory layout fits, i.e. not for dilated windows)
constexpr int kPairStaged = 4;
// TcLaunch::flags bit: the launch's input is relu(plane) -- two ReLU warps per CTA apply it to each
// window stage in shared memory before the UMMAs read it (MRB blocks' conv1: the previous conv2 then
// writes one plane instead of a second, pre-activated copy).  Every group of the launch has it.
constexpr int kPairReluIn = 8;

// True for a 3x3 96 -> 96 conv whose window (halo rows either side) fits the pair kernel's smem.
bool conv_pair96_supported(int cin, int cout, int ks, int halo);
// Window pipeline depth that fits in shared memory for `win_alloc`-row windows (0: none); `staged`:
// a launch with a residual or a second output (TMA-staged epilogue).
int conv_pair96_stages(int win_alloc, bool staged);
size_t conv_pair96_smem_bytes(int stages, int win_alloc, bool staged);
// Grid: CTA pairs (cluster of 2), at most num_sms / 2 pairs.  Returns the kernel name.
const char* conv_pair96_launch(const TcLaunch& L, int num_sms, cudaStream_t stream);

}  // namespace cnrx
