// Single translation unit of libjv.so (one TU keeps the device-side hang
// flag and the launch helper shared without relocatable device code).
#include "abi.cu"
#include "spmv.cu"
#include "factor.cu"
#include "solve.cu"
#include "setup.cu"
#include "rcm.cu"
#include "elim.cu"
#include "tail.cu"
#include "region.cu"
#include "regions_host.cpp"
#include "blas.cu"
#include "host.cpp"
