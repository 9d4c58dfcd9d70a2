// ABI version / metadata entry points.
#include "common.cuh"

extern "C" int sst_abi_version(void) { return SST_ABI_VERSION; }
