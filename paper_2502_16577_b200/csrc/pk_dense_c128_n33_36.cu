// Instantiates the dense complex register kernel for orders 33..36.
#include "pk_dense_c128_launch.cuh"
PK_INSTANTIATE_DENSE_C128(33)
PK_INSTANTIATE_DENSE_C128(34)
PK_INSTANTIATE_DENSE_C128(35)
PK_INSTANTIATE_DENSE_C128(36)
