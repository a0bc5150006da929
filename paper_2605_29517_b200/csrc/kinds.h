// Operand kinds of the tensor-core kernels (shared by device headers and host launchers).
#pragma once

namespace mxs {
enum class TcKind : int { BF16 = 0, F16 = 1, I8 = 2 };
}  // namespace mxs
