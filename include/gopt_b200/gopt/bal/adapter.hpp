// Drop-in path shim: the reference header gopt/bal/adapter.hpp maps onto the B200 facade.
#pragma once
#include "../../gopt.hpp"
