// Instantiates the exact integer register kernel for orders 54..58.
#include "pk_int_launch.cuh"
PK_INSTANTIATE_INT(54)
PK_INSTANTIATE_INT(55)
PK_INSTANTIATE_INT(56)
PK_INSTANTIATE_INT(57)
PK_INSTANTIATE_INT(58)
