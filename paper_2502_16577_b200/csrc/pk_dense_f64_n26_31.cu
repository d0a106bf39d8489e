// Instantiates the dense real register kernel for orders 26..31 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(26)
PK_INSTANTIATE_DENSE_F64(27)
PK_INSTANTIATE_DENSE_F64(28)
PK_INSTANTIATE_DENSE_F64(29)
PK_INSTANTIATE_DENSE_F64(30)
PK_INSTANTIATE_DENSE_F64(31)
