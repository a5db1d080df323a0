# Top-level build. `make` builds the sm_100a product library, the host-only
# synthetic-data library, the CPU oracle (+ reference shim when
# /root/reference exists) and the C++ test binaries.
NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG      := paper_1403_1706_b200
CSRC     := $(PKG)/csrc
CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(CU_SRCS))
LIB      := $(PKG)/libqgm_b200.so
SYNTH    := $(PKG)/libqgm_synth.so
HOSTFLAGS := -O3 -march=x86-64-v3 -std=c++20 -pthread -fPIC -Wall
CPP_TESTS := $(patsubst tests/cpp/%.cpp,tests/cpp/build/%,$(filter-out tests/cpp/catch_main.cpp,$(wildcard tests/cpp/test_*.cpp)))

.PHONY: all lib oracle tests clean
all: lib oracle tests
lib: $(LIB) $(SYNTH)

build/obj/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) $(CSRC)/internal.hpp include/qgm_c.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

$(LIB): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^

$(SYNTH): $(CSRC)/synth.cpp
	$(CXX) $(HOSTFLAGS) -shared -o $@ $<

oracle:
	$(MAKE) -C oracle

tests: $(CPP_TESTS)

tests/cpp/build/%: tests/cpp/%.cpp tests/cpp/catch_main.cpp tests/cpp/catch2/catch_amalgamated.hpp $(wildcard include/qgmap/*.hpp) include/qgm_c.h $(LIB)
	@mkdir -p $(dir $@)
	$(CXX) $(HOSTFLAGS) -Iinclude -Itests/cpp -Ioracle -o $@ $< tests/cpp/catch_main.cpp -L$(PKG) -lqgm_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

tools/run_map_bench: tools/run_map_bench.cpp $(wildcard include/qgmap/*.hpp) include/qgm_c.h $(LIB)
	$(CXX) $(HOSTFLAGS) -Iinclude -o $@ $< -L$(PKG) -lqgm_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

clean:
	rm -rf build tests/cpp/build $(LIB) $(SYNTH) tools/run_map_bench
	$(MAKE) -C oracle clean
