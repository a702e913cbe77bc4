// forwarding header: the reference include path lowprec/quantize.hpp served by the B200 shim
#pragma once
#include "lowprec_shim.hpp"
