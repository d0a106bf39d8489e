// Instantiates the dense real register kernel for orders 46..49 (split for parallel builds).
#include "pk_dense_f64_launch.cuh"
PK_INSTANTIATE_DENSE_F64(46)
PK_INSTANTIATE_DENSE_F64(47)
PK_INSTANTIATE_DENSE_F64(48)
PK_INSTANTIATE_DENSE_F64(49)
