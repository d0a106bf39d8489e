// Instantiates the exact integer register kernel for orders 48..53.
#include "pk_int_launch.cuh"
PK_INSTANTIATE_INT(48)
PK_INSTANTIATE_INT(49)
PK_INSTANTIATE_INT(50)
PK_INSTANTIATE_INT(51)
PK_INSTANTIATE_INT(52)
PK_INSTANTIATE_INT(53)
