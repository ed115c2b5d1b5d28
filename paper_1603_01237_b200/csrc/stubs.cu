// stubs.cu — kinds whose device kernels are not built yet report "not supported".
#include "kernels.h"

namespace qoc {
cudaError_t strang_task(const DevProblem&, const DevRun&, const TaskArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t strang_horizon(const DevProblem&, const DevRun&, int, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace qoc
