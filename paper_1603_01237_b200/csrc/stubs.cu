// stubs.cu — kinds whose device kernels are not built yet report "not supported".
#include "kernels.h"

namespace qoc {
}  // namespace qoc
