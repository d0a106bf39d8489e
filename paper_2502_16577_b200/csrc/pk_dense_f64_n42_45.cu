// Instantiates the dense real register kernel for orders 42..45 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(42)
PK_INSTANTIATE_DENSE_F64(43)
PK_INSTANTIATE_DENSE_F64(44)
PK_INSTANTIATE_DENSE_F64(45)
