// Instantiates the dense real register kernel for orders 50..53 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(50)
PK_INSTANTIATE_DENSE_F64(51)
PK_INSTANTIATE_DENSE_F64(52)
PK_INSTANTIATE_DENSE_F64(53)
