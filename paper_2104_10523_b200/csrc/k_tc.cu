// a7 (tensor-core path): placeholder until the tcgen05 / DMMA kernels land.
#include "kernels.hpp"

namespace tnqvm {
namespace dev {

size_t tc_wbuf_bytes(int, int) { return 0; }
bool tc_supported(int, int) { return false; }
void launch_gemm_tc(const GemmDesc&, void*, cudaStream_t) {}
bool dmma_supported(int, int) { return false; }
void launch_gemm_dmma(const GemmDesc&, cudaStream_t) {}

}  // namespace dev
}  // namespace tnqvm
