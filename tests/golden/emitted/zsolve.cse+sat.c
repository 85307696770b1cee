void z_solve_lhs(double fjacZ[5][5][258][258][258], double njacZ[5][5][258][258][258], double lhsZ[5][5][3][258][258][258], double dt, double tz1, double tz2, double dz1, double dz2, double dz3, double dz4, double dz5, int kbeg, int kend, int ny, int nx) {
    int k, i, j;
    double temp1, temp2;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop worker
        for (i = 1; i < ny - 1; i++) {
            #pragma acc loop vector
            for (j = 1; j < nx - 1; j++) {
                double _v2;
                _v2 = dt * tz1;
                temp1 = _v2;
                {
                    double _v4;
                    _v4 = dt * tz2;
                    temp2 = _v4;
                    {
                        int _v11;
                        double _v12, _v14, _v9, _v13, _v15, _v16, _v18, _v19;
                        _v11 = k - 1;
                        _v12 = fjacZ[0][0][_v11][i][j];
                        _v14 = njacZ[0][0][_v11][i][j];
                        _v9 = -_v4;
                        _v13 = _v9 * _v12;
                        _v15 = _v2 * _v14;
                        _v16 = _v13 - _v15;
                        _v18 = _v2 * dz1;
                        _v19 = _v16 - _v18;
                        lhsZ[0][0][0][k][i][j] = _v19;
                        {
                            double _v20, _v22, _v21, _v23, _v24;
                            _v20 = fjacZ[0][1][_v11][i][j];
                            _v22 = njacZ[0][1][_v11][i][j];
                            _v21 = _v9 * _v20;
                            _v23 = _v2 * _v22;
                            _v24 = _v21 - _v23;
                            lhsZ[0][1][0][k][i][j] = _v24;
                            {
                                double _v26, _v28, _v27, _v29, _v30;
                                _v26 = fjacZ[0][2][_v11][i][j];
                                _v28 = njacZ[0][2][_v11][i][j];
                                _v27 = _v9 * _v26;
                                _v29 = _v2 * _v28;
                                _v30 = _v27 - _v29;
                                lhsZ[0][2][0][k][i][j] = _v30;
                                {
                                    double _v32, _v34, _v33, _v35, _v36;
                                    _v32 = fjacZ[0][3][_v11][i][j];
                                    _v34 = njacZ[0][3][_v11][i][j];
                                    _v33 = _v9 * _v32;
                                    _v35 = _v2 * _v34;
                                    _v36 = _v33 - _v35;
                                    lhsZ[0][3][0][k][i][j] = _v36;
                                    {
                                        double _v38, _v40, _v39, _v41, _v42;
                                        _v38 = fjacZ[0][4][_v11][i][j];
                                        _v40 = njacZ[0][4][_v11][i][j];
                                        _v39 = _v9 * _v38;
                                        _v41 = _v2 * _v40;
                                        _v42 = _v39 - _v41;
                                        lhsZ[0][4][0][k][i][j] = _v42;
                                        {
                                            double _v43, _v45, _v44, _v46, _v47;
                                            _v43 = fjacZ[1][0][_v11][i][j];
                                            _v45 = njacZ[1][0][_v11][i][j];
                                            _v44 = _v9 * _v43;
                                            _v46 = _v2 * _v45;
                                            _v47 = _v44 - _v46;
                                            lhsZ[1][0][0][k][i][j] = _v47;
                                            {
                                                double _v48, _v50, _v49, _v51, _v52, _v54, _v55;
                                                _v48 = fjacZ[1][1][_v11][i][j];
                                                _v50 = njacZ[1][1][_v11][i][j];
                                                _v49 = _v9 * _v48;
                                                _v51 = _v2 * _v50;
                                                _v52 = _v49 - _v51;
                                                _v54 = _v2 * dz2;
                                                _v55 = _v52 - _v54;
                                                lhsZ[1][1][0][k][i][j] = _v55;
                                                {
                                                    double _v56, _v58, _v57, _v59, _v60;
                                                    _v56 = fjacZ[1][2][_v11][i][j];
                                                    _v58 = njacZ[1][2][_v11][i][j];
                                                    _v57 = _v9 * _v56;
                                                    _v59 = _v2 * _v58;
                                                    _v60 = _v57 - _v59;
                                                    lhsZ[1][2][0][k][i][j] = _v60;
                                                    {
                                                        double _v61, _v63, _v62, _v64, _v65;
                                                        _v61 = fjacZ[1][3][_v11][i][j];
                                                        _v63 = njacZ[1][3][_v11][i][j];
                                                        _v62 = _v9 * _v61;
                                                        _v64 = _v2 * _v63;
                                                        _v65 = _v62 - _v64;
                                                        lhsZ[1][3][0][k][i][j] = _v65;
                                                        {
                                                            double _v66, _v68, _v67, _v69, _v70;
                                                            _v66 = fjacZ[1][4][_v11][i][j];
                                                            _v68 = njacZ[1][4][_v11][i][j];
                                                            _v67 = _v9 * _v66;
                                                            _v69 = _v2 * _v68;
                                                            _v70 = _v67 - _v69;
                                                            lhsZ[1][4][0][k][i][j] = _v70;
                                                            {
                                                                double _v71, _v73, _v72, _v74, _v75;
                                                                _v71 = fjacZ[2][0][_v11][i][j];
                                                                _v73 = njacZ[2][0][_v11][i][j];
                                                                _v72 = _v9 * _v71;
                                                                _v74 = _v2 * _v73;
                                                                _v75 = _v72 - _v74;
                                                                lhsZ[2][0][0][k][i][j] = _v75;
                                                                {
                                                                    double _v76, _v78, _v77, _v79, _v80;
                                                                    _v76 = fjacZ[2][1][_v11][i][j];
                                                                    _v78 = njacZ[2][1][_v11][i][j];
                                                                    _v77 = _v9 * _v76;
                                                                    _v79 = _v2 * _v78;
                                                                    _v80 = _v77 - _v79;
                                                                    lhsZ[2][1][0][k][i][j] = _v80;
                                                                    {
                                                                        double _v81, _v83, _v82, _v84, _v85, _v87, _v88;
                                                                        _v81 = fjacZ[2][2][_v11][i][j];
                                                                        _v83 = njacZ[2][2][_v11][i][j];
                                                                        _v82 = _v9 * _v81;
                                                                        _v84 = _v2 * _v83;
                                                                        _v85 = _v82 - _v84;
                                                                        _v87 = _v2 * dz3;
                                                                        _v88 = _v85 - _v87;
                                                                        lhsZ[2][2][0][k][i][j] = _v88;
                                                                        {
                                                                            double _v89, _v91, _v90, _v92, _v93;
                                                                            _v89 = fjacZ[2][3][_v11][i][j];
                                                                            _v91 = njacZ[2][3][_v11][i][j];
                                                                            _v90 = _v9 * _v89;
                                                                            _v92 = _v2 * _v91;
                                                                            _v93 = _v90 - _v92;
                                                                            lhsZ[2][3][0][k][i][j] = _v93;
                                                                            {
                                                                                double _v94, _v96, _v95, _v97, _v98;
                                                                                _v94 = fjacZ[2][4][_v11][i][j];
                                                                                _v96 = njacZ[2][4][_v11][i][j];
                                                                                _v95 = _v9 * _v94;
                                                                                _v97 = _v2 * _v96;
                                                                                _v98 = _v95 - _v97;
                                                                                lhsZ[2][4][0][k][i][j] = _v98;
                                                                                {
                                                                                    double _v99, _v101, _v100, _v102, _v103;
                                                                                    _v99 = fjacZ[3][0][_v11][i][j];
                                                                                    _v101 = njacZ[3][0][_v11][i][j];
                                                                                    _v100 = _v9 * _v99;
                                                                                    _v102 = _v2 * _v101;
                                                                                    _v103 = _v100 - _v102;
                                                                                    lhsZ[3][0][0][k][i][j] = _v103;
                                                                                    {
                                                                                        double _v104, _v106, _v105, _v107, _v108;
                                                                                        _v104 = fjacZ[3][1][_v11][i][j];
                                                                                        _v106 = njacZ[3][1][_v11][i][j];
                                                                                        _v105 = _v9 * _v104;
                                                                                        _v107 = _v2 * _v106;
                                                                                        _v108 = _v105 - _v107;
                                                                                        lhsZ[3][1][0][k][i][j] = _v108;
                                                                                        {
                                                                                            double _v109, _v111, _v110, _v112, _v113;
                                                                                            _v109 = fjacZ[3][2][_v11][i][j];
                                                                                            _v111 = njacZ[3][2][_v11][i][j];
                                                                                            _v110 = _v9 * _v109;
                                                                                            _v112 = _v2 * _v111;
                                                                                            _v113 = _v110 - _v112;
                                                                                            lhsZ[3][2][0][k][i][j] = _v113;
                                                                                            {
                                                                                                double _v114, _v116, _v115, _v117, _v118, _v120, _v121;
                                                                                                _v114 = fjacZ[3][3][_v11][i][j];
                                                                                                _v116 = njacZ[3][3][_v11][i][j];
                                                                                                _v115 = _v9 * _v114;
                                                                                                _v117 = _v2 * _v116;
                                                                                                _v118 = _v115 - _v117;
                                                                                                _v120 = _v2 * dz4;
                                                                                                _v121 = _v118 - _v120;
                                                                                                lhsZ[3][3][0][k][i][j] = _v121;
                                                                                                {
                                                                                                    double _v122, _v124, _v123, _v125, _v126;
                                                                                                    _v122 = fjacZ[3][4][_v11][i][j];
                                                                                                    _v124 = njacZ[3][4][_v11][i][j];
                                                                                                    _v123 = _v9 * _v122;
                                                                                                    _v125 = _v2 * _v124;
                                                                                                    _v126 = _v123 - _v125;
                                                                                                    lhsZ[3][4][0][k][i][j] = _v126;
                                                                                                    {
                                                                                                        double _v127, _v129, _v128, _v130, _v131;
                                                                                                        _v127 = fjacZ[4][0][_v11][i][j];
                                                                                                        _v129 = njacZ[4][0][_v11][i][j];
                                                                                                        _v128 = _v9 * _v127;
                                                                                                        _v130 = _v2 * _v129;
                                                                                                        _v131 = _v128 - _v130;
                                                                                                        lhsZ[4][0][0][k][i][j] = _v131;
                                                                                                        {
                                                                                                            double _v132, _v134, _v133, _v135, _v136;
                                                                                                            _v132 = fjacZ[4][1][_v11][i][j];
                                                                                                            _v134 = njacZ[4][1][_v11][i][j];
                                                                                                            _v133 = _v9 * _v132;
                                                                                                            _v135 = _v2 * _v134;
                                                                                                            _v136 = _v133 - _v135;
                                                                                                            lhsZ[4][1][0][k][i][j] = _v136;
                                                                                                            {
                                                                                                                double _v137, _v139, _v138, _v140, _v141;
                                                                                                                _v137 = fjacZ[4][2][_v11][i][j];
                                                                                                                _v139 = njacZ[4][2][_v11][i][j];
                                                                                                                _v138 = _v9 * _v137;
                                                                                                                _v140 = _v2 * _v139;
                                                                                                                _v141 = _v138 - _v140;
                                                                                                                lhsZ[4][2][0][k][i][j] = _v141;
                                                                                                                {
                                                                                                                    double _v142, _v144, _v143, _v145, _v146;
                                                                                                                    _v142 = fjacZ[4][3][_v11][i][j];
                                                                                                                    _v144 = njacZ[4][3][_v11][i][j];
                                                                                                                    _v143 = _v9 * _v142;
                                                                                                                    _v145 = _v2 * _v144;
                                                                                                                    _v146 = _v143 - _v145;
                                                                                                                    lhsZ[4][3][0][k][i][j] = _v146;
                                                                                                                    {
                                                                                                                        double _v147, _v149, _v148, _v150, _v151, _v153, _v154;
                                                                                                                        _v147 = fjacZ[4][4][_v11][i][j];
                                                                                                                        _v149 = njacZ[4][4][_v11][i][j];
                                                                                                                        _v148 = _v9 * _v147;
                                                                                                                        _v150 = _v2 * _v149;
                                                                                                                        _v151 = _v148 - _v150;
                                                                                                                        _v153 = _v2 * dz5;
                                                                                                                        _v154 = _v151 - _v153;
                                                                                                                        lhsZ[4][4][0][k][i][j] = _v154;
                                                                                                                        {
                                                                                                                            double _v158, _v157, _v160, _v162;
                                                                                                                            _v158 = njacZ[0][0][k][i][j];
                                                                                                                            _v157 = _v2 * 2.0;
                                                                                                                            _v160 = 1.0 + _v157 * _v158;
                                                                                                                            _v162 = _v160 + _v157 * dz1;
                                                                                                                            lhsZ[0][0][1][k][i][j] = _v162;
                                                                                                                            {
                                                                                                                                double _v163, _v164;
                                                                                                                                _v163 = njacZ[0][1][k][i][j];
                                                                                                                                _v164 = _v157 * _v163;
                                                                                                                                lhsZ[0][1][1][k][i][j] = _v164;
                                                                                                                                {
                                                                                                                                    double _v165, _v166;
                                                                                                                                    _v165 = njacZ[0][2][k][i][j];
                                                                                                                                    _v166 = _v157 * _v165;
                                                                                                                                    lhsZ[0][2][1][k][i][j] = _v166;
                                                                                                                                    {
                                                                                                                                        double _v167, _v168;
                                                                                                                                        _v167 = njacZ[0][3][k][i][j];
                                                                                                                                        _v168 = _v157 * _v167;
                                                                                                                                        lhsZ[0][3][1][k][i][j] = _v168;
                                                                                                                                        {
                                                                                                                                            double _v169, _v170;
                                                                                                                                            _v169 = njacZ[0][4][k][i][j];
                                                                                                                                            _v170 = _v157 * _v169;
                                                                                                                                            lhsZ[0][4][1][k][i][j] = _v170;
                                                                                                                                            {
                                                                                                                                                double _v171, _v172;
                                                                                                                                                _v171 = njacZ[1][0][k][i][j];
                                                                                                                                                _v172 = _v157 * _v171;
                                                                                                                                                lhsZ[1][0][1][k][i][j] = _v172;
                                                                                                                                                {
                                                                                                                                                    double _v173, _v175, _v177;
                                                                                                                                                    _v173 = njacZ[1][1][k][i][j];
                                                                                                                                                    _v175 = 1.0 + _v157 * _v173;
                                                                                                                                                    _v177 = _v175 + _v157 * dz2;
                                                                                                                                                    lhsZ[1][1][1][k][i][j] = _v177;
                                                                                                                                                    {
                                                                                                                                                        double _v178, _v179;
                                                                                                                                                        _v178 = njacZ[1][2][k][i][j];
                                                                                                                                                        _v179 = _v157 * _v178;
                                                                                                                                                        lhsZ[1][2][1][k][i][j] = _v179;
                                                                                                                                                        {
                                                                                                                                                            double _v180, _v181;
                                                                                                                                                            _v180 = njacZ[1][3][k][i][j];
                                                                                                                                                            _v181 = _v157 * _v180;
                                                                                                                                                            lhsZ[1][3][1][k][i][j] = _v181;
                                                                                                                                                            {
                                                                                                                                                                double _v182, _v183;
                                                                                                                                                                _v182 = njacZ[1][4][k][i][j];
                                                                                                                                                                _v183 = _v157 * _v182;
                                                                                                                                                                lhsZ[1][4][1][k][i][j] = _v183;
                                                                                                                                                                {
                                                                                                                                                                    double _v184, _v185;
                                                                                                                                                                    _v184 = njacZ[2][0][k][i][j];
                                                                                                                                                                    _v185 = _v157 * _v184;
                                                                                                                                                                    lhsZ[2][0][1][k][i][j] = _v185;
                                                                                                                                                                    {
                                                                                                                                                                        double _v186, _v187;
                                                                                                                                                                        _v186 = njacZ[2][1][k][i][j];
                                                                                                                                                                        _v187 = _v157 * _v186;
                                                                                                                                                                        lhsZ[2][1][1][k][i][j] = _v187;
                                                                                                                                                                        {
                                                                                                                                                                            double _v188, _v190, _v192;
                                                                                                                                                                            _v188 = njacZ[2][2][k][i][j];
                                                                                                                                                                            _v190 = 1.0 + _v157 * _v188;
                                                                                                                                                                            _v192 = _v190 + _v157 * dz3;
                                                                                                                                                                            lhsZ[2][2][1][k][i][j] = _v192;
                                                                                                                                                                            {
                                                                                                                                                                                double _v193, _v194;
                                                                                                                                                                                _v193 = njacZ[2][3][k][i][j];
                                                                                                                                                                                _v194 = _v157 * _v193;
                                                                                                                                                                                lhsZ[2][3][1][k][i][j] = _v194;
                                                                                                                                                                                {
                                                                                                                                                                                    double _v195, _v196;
                                                                                                                                                                                    _v195 = njacZ[2][4][k][i][j];
                                                                                                                                                                                    _v196 = _v157 * _v195;
                                                                                                                                                                                    lhsZ[2][4][1][k][i][j] = _v196;
                                                                                                                                                                                    {
                                                                                                                                                                                        double _v197, _v198;
                                                                                                                                                                                        _v197 = njacZ[3][0][k][i][j];
                                                                                                                                                                                        _v198 = _v157 * _v197;
                                                                                                                                                                                        lhsZ[3][0][1][k][i][j] = _v198;
                                                                                                                                                                                        {
                                                                                                                                                                                            double _v199, _v200;
                                                                                                                                                                                            _v199 = njacZ[3][1][k][i][j];
                                                                                                                                                                                            _v200 = _v157 * _v199;
                                                                                                                                                                                            lhsZ[3][1][1][k][i][j] = _v200;
                                                                                                                                                                                            {
                                                                                                                                                                                                double _v201, _v202;
                                                                                                                                                                                                _v201 = njacZ[3][2][k][i][j];
                                                                                                                                                                                                _v202 = _v157 * _v201;
                                                                                                                                                                                                lhsZ[3][2][1][k][i][j] = _v202;
                                                                                                                                                                                                {
                                                                                                                                                                                                    double _v203, _v205, _v207;
                                                                                                                                                                                                    _v203 = njacZ[3][3][k][i][j];
                                                                                                                                                                                                    _v205 = 1.0 + _v157 * _v203;
                                                                                                                                                                                                    _v207 = _v205 + _v157 * dz4;
                                                                                                                                                                                                    lhsZ[3][3][1][k][i][j] = _v207;
                                                                                                                                                                                                    {
                                                                                                                                                                                                        double _v208, _v209;
                                                                                                                                                                                                        _v208 = njacZ[3][4][k][i][j];
                                                                                                                                                                                                        _v209 = _v157 * _v208;
                                                                                                                                                                                                        lhsZ[3][4][1][k][i][j] = _v209;
                                                                                                                                                                                                        {
                                                                                                                                                                                                            double _v210, _v211;
                                                                                                                                                                                                            _v210 = njacZ[4][0][k][i][j];
                                                                                                                                                                                                            _v211 = _v157 * _v210;
                                                                                                                                                                                                            lhsZ[4][0][1][k][i][j] = _v211;
                                                                                                                                                                                                            {
                                                                                                                                                                                                                double _v212, _v213;
                                                                                                                                                                                                                _v212 = njacZ[4][1][k][i][j];
                                                                                                                                                                                                                _v213 = _v157 * _v212;
                                                                                                                                                                                                                lhsZ[4][1][1][k][i][j] = _v213;
                                                                                                                                                                                                                {
                                                                                                                                                                                                                    double _v214, _v215;
                                                                                                                                                                                                                    _v214 = njacZ[4][2][k][i][j];
                                                                                                                                                                                                                    _v215 = _v157 * _v214;
                                                                                                                                                                                                                    lhsZ[4][2][1][k][i][j] = _v215;
                                                                                                                                                                                                                    {
                                                                                                                                                                                                                        double _v216, _v217;
                                                                                                                                                                                                                        _v216 = njacZ[4][3][k][i][j];
                                                                                                                                                                                                                        _v217 = _v157 * _v216;
                                                                                                                                                                                                                        lhsZ[4][3][1][k][i][j] = _v217;
                                                                                                                                                                                                                        {
                                                                                                                                                                                                                            double _v218, _v220, _v222;
                                                                                                                                                                                                                            _v218 = njacZ[4][4][k][i][j];
                                                                                                                                                                                                                            _v220 = 1.0 + _v157 * _v218;
                                                                                                                                                                                                                            _v222 = _v220 + _v157 * dz5;
                                                                                                                                                                                                                            lhsZ[4][4][1][k][i][j] = _v222;
                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                int _v223;
                                                                                                                                                                                                                                double _v224, _v226, _v225, _v227, _v228, _v229;
                                                                                                                                                                                                                                _v223 = k + 1;
                                                                                                                                                                                                                                _v224 = fjacZ[0][0][_v223][i][j];
                                                                                                                                                                                                                                _v226 = njacZ[0][0][_v223][i][j];
                                                                                                                                                                                                                                _v225 = _v4 * _v224;
                                                                                                                                                                                                                                _v227 = _v2 * _v226;
                                                                                                                                                                                                                                _v228 = _v225 - _v227;
                                                                                                                                                                                                                                _v229 = _v228 - _v18;
                                                                                                                                                                                                                                lhsZ[0][0][2][k][i][j] = _v229;
                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                    double _v230, _v232, _v231, _v233, _v234;
                                                                                                                                                                                                                                    _v230 = fjacZ[0][1][_v223][i][j];
                                                                                                                                                                                                                                    _v232 = njacZ[0][1][_v223][i][j];
                                                                                                                                                                                                                                    _v231 = _v4 * _v230;
                                                                                                                                                                                                                                    _v233 = _v2 * _v232;
                                                                                                                                                                                                                                    _v234 = _v231 - _v233;
                                                                                                                                                                                                                                    lhsZ[0][1][2][k][i][j] = _v234;
                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                        double _v235, _v237, _v236, _v238, _v239;
                                                                                                                                                                                                                                        _v235 = fjacZ[0][2][_v223][i][j];
                                                                                                                                                                                                                                        _v237 = njacZ[0][2][_v223][i][j];
                                                                                                                                                                                                                                        _v236 = _v4 * _v235;
                                                                                                                                                                                                                                        _v238 = _v2 * _v237;
                                                                                                                                                                                                                                        _v239 = _v236 - _v238;
                                                                                                                                                                                                                                        lhsZ[0][2][2][k][i][j] = _v239;
                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                            double _v240, _v242, _v241, _v243, _v244;
                                                                                                                                                                                                                                            _v240 = fjacZ[0][3][_v223][i][j];
                                                                                                                                                                                                                                            _v242 = njacZ[0][3][_v223][i][j];
                                                                                                                                                                                                                                            _v241 = _v4 * _v240;
                                                                                                                                                                                                                                            _v243 = _v2 * _v242;
                                                                                                                                                                                                                                            _v244 = _v241 - _v243;
                                                                                                                                                                                                                                            lhsZ[0][3][2][k][i][j] = _v244;
                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                double _v245, _v247, _v246, _v248, _v249;
                                                                                                                                                                                                                                                _v245 = fjacZ[0][4][_v223][i][j];
                                                                                                                                                                                                                                                _v247 = njacZ[0][4][_v223][i][j];
                                                                                                                                                                                                                                                _v246 = _v4 * _v245;
                                                                                                                                                                                                                                                _v248 = _v2 * _v247;
                                                                                                                                                                                                                                                _v249 = _v246 - _v248;
                                                                                                                                                                                                                                                lhsZ[0][4][2][k][i][j] = _v249;
                                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                                    double _v250, _v252, _v251, _v253, _v254;
                                                                                                                                                                                                                                                    _v250 = fjacZ[1][0][_v223][i][j];
                                                                                                                                                                                                                                                    _v252 = njacZ[1][0][_v223][i][j];
                                                                                                                                                                                                                                                    _v251 = _v4 * _v250;
                                                                                                                                                                                                                                                    _v253 = _v2 * _v252;
                                                                                                                                                                                                                                                    _v254 = _v251 - _v253;
                                                                                                                                                                                                                                                    lhsZ[1][0][2][k][i][j] = _v254;
                                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                                        double _v255, _v257, _v256, _v258, _v259, _v260;
                                                                                                                                                                                                                                                        _v255 = fjacZ[1][1][_v223][i][j];
                                                                                                                                                                                                                                                        _v257 = njacZ[1][1][_v223][i][j];
                                                                                                                                                                                                                                                        _v256 = _v4 * _v255;
                                                                                                                                                                                                                                                        _v258 = _v2 * _v257;
                                                                                                                                                                                                                                                        _v259 = _v256 - _v258;
                                                                                                                                                                                                                                                        _v260 = _v259 - _v54;
                                                                                                                                                                                                                                                        lhsZ[1][1][2][k][i][j] = _v260;
                                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                                            double _v261, _v263, _v262, _v264, _v265;
                                                                                                                                                                                                                                                            _v261 = fjacZ[1][2][_v223][i][j];
                                                                                                                                                                                                                                                            _v263 = njacZ[1][2][_v223][i][j];
                                                                                                                                                                                                                                                            _v262 = _v4 * _v261;
                                                                                                                                                                                                                                                            _v264 = _v2 * _v263;
                                                                                                                                                                                                                                                            _v265 = _v262 - _v264;
                                                                                                                                                                                                                                                            lhsZ[1][2][2][k][i][j] = _v265;
                                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                                double _v266, _v268, _v267, _v269, _v270;
                                                                                                                                                                                                                                                                _v266 = fjacZ[1][3][_v223][i][j];
                                                                                                                                                                                                                                                                _v268 = njacZ[1][3][_v223][i][j];
                                                                                                                                                                                                                                                                _v267 = _v4 * _v266;
                                                                                                                                                                                                                                                                _v269 = _v2 * _v268;
                                                                                                                                                                                                                                                                _v270 = _v267 - _v269;
                                                                                                                                                                                                                                                                lhsZ[1][3][2][k][i][j] = _v270;
                                                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                                                    double _v271, _v273, _v272, _v274, _v275;
                                                                                                                                                                                                                                                                    _v271 = fjacZ[1][4][_v223][i][j];
                                                                                                                                                                                                                                                                    _v273 = njacZ[1][4][_v223][i][j];
                                                                                                                                                                                                                                                                    _v272 = _v4 * _v271;
                                                                                                                                                                                                                                                                    _v274 = _v2 * _v273;
                                                                                                                                                                                                                                                                    _v275 = _v272 - _v274;
                                                                                                                                                                                                                                                                    lhsZ[1][4][2][k][i][j] = _v275;
                                                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                                                        double _v276, _v278, _v277, _v279, _v280;
                                                                                                                                                                                                                                                                        _v276 = fjacZ[2][0][_v223][i][j];
                                                                                                                                                                                                                                                                        _v278 = njacZ[2][0][_v223][i][j];
                                                                                                                                                                                                                                                                        _v277 = _v4 * _v276;
                                                                                                                                                                                                                                                                        _v279 = _v2 * _v278;
                                                                                                                                                                                                                                                                        _v280 = _v277 - _v279;
                                                                                                                                                                                                                                                                        lhsZ[2][0][2][k][i][j] = _v280;
                                                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                                                            double _v281, _v283, _v282, _v284, _v285;
                                                                                                                                                                                                                                                                            _v281 = fjacZ[2][1][_v223][i][j];
                                                                                                                                                                                                                                                                            _v283 = njacZ[2][1][_v223][i][j];
                                                                                                                                                                                                                                                                            _v282 = _v4 * _v281;
                                                                                                                                                                                                                                                                            _v284 = _v2 * _v283;
                                                                                                                                                                                                                                                                            _v285 = _v282 - _v284;
                                                                                                                                                                                                                                                                            lhsZ[2][1][2][k][i][j] = _v285;
                                                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                                                double _v286, _v288, _v287, _v289, _v290, _v291;
                                                                                                                                                                                                                                                                                _v286 = fjacZ[2][2][_v223][i][j];
                                                                                                                                                                                                                                                                                _v288 = njacZ[2][2][_v223][i][j];
                                                                                                                                                                                                                                                                                _v287 = _v4 * _v286;
                                                                                                                                                                                                                                                                                _v289 = _v2 * _v288;
                                                                                                                                                                                                                                                                                _v290 = _v287 - _v289;
                                                                                                                                                                                                                                                                                _v291 = _v290 - _v87;
                                                                                                                                                                                                                                                                                lhsZ[2][2][2][k][i][j] = _v291;
                                                                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                                                                    double _v292, _v294, _v293, _v295, _v296;
                                                                                                                                                                                                                                                                                    _v292 = fjacZ[2][3][_v223][i][j];
                                                                                                                                                                                                                                                                                    _v294 = njacZ[2][3][_v223][i][j];
                                                                                                                                                                                                                                                                                    _v293 = _v4 * _v292;
                                                                                                                                                                                                                                                                                    _v295 = _v2 * _v294;
                                                                                                                                                                                                                                                                                    _v296 = _v293 - _v295;
                                                                                                                                                                                                                                                                                    lhsZ[2][3][2][k][i][j] = _v296;
                                                                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                                                                        double _v297, _v299, _v298, _v300, _v301;
                                                                                                                                                                                                                                                                                        _v297 = fjacZ[2][4][_v223][i][j];
                                                                                                                                                                                                                                                                                        _v299 = njacZ[2][4][_v223][i][j];
                                                                                                                                                                                                                                                                                        _v298 = _v4 * _v297;
                                                                                                                                                                                                                                                                                        _v300 = _v2 * _v299;
                                                                                                                                                                                                                                                                                        _v301 = _v298 - _v300;
                                                                                                                                                                                                                                                                                        lhsZ[2][4][2][k][i][j] = _v301;
                                                                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                                                                            double _v302, _v304, _v303, _v305, _v306;
                                                                                                                                                                                                                                                                                            _v302 = fjacZ[3][0][_v223][i][j];
                                                                                                                                                                                                                                                                                            _v304 = njacZ[3][0][_v223][i][j];
                                                                                                                                                                                                                                                                                            _v303 = _v4 * _v302;
                                                                                                                                                                                                                                                                                            _v305 = _v2 * _v304;
                                                                                                                                                                                                                                                                                            _v306 = _v303 - _v305;
                                                                                                                                                                                                                                                                                            lhsZ[3][0][2][k][i][j] = _v306;
                                                                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                                                                double _v307, _v309, _v308, _v310, _v311;
                                                                                                                                                                                                                                                                                                _v307 = fjacZ[3][1][_v223][i][j];
                                                                                                                                                                                                                                                                                                _v309 = njacZ[3][1][_v223][i][j];
                                                                                                                                                                                                                                                                                                _v308 = _v4 * _v307;
                                                                                                                                                                                                                                                                                                _v310 = _v2 * _v309;
                                                                                                                                                                                                                                                                                                _v311 = _v308 - _v310;
                                                                                                                                                                                                                                                                                                lhsZ[3][1][2][k][i][j] = _v311;
                                                                                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                                                                                    double _v312, _v314, _v313, _v315, _v316;
                                                                                                                                                                                                                                                                                                    _v312 = fjacZ[3][2][_v223][i][j];
                                                                                                                                                                                                                                                                                                    _v314 = njacZ[3][2][_v223][i][j];
                                                                                                                                                                                                                                                                                                    _v313 = _v4 * _v312;
                                                                                                                                                                                                                                                                                                    _v315 = _v2 * _v314;
                                                                                                                                                                                                                                                                                                    _v316 = _v313 - _v315;
                                                                                                                                                                                                                                                                                                    lhsZ[3][2][2][k][i][j] = _v316;
                                                                                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                                                                                        double _v317, _v319, _v318, _v320, _v321, _v322;
                                                                                                                                                                                                                                                                                                        _v317 = fjacZ[3][3][_v223][i][j];
                                                                                                                                                                                                                                                                                                        _v319 = njacZ[3][3][_v223][i][j];
                                                                                                                                                                                                                                                                                                        _v318 = _v4 * _v317;
                                                                                                                                                                                                                                                                                                        _v320 = _v2 * _v319;
                                                                                                                                                                                                                                                                                                        _v321 = _v318 - _v320;
                                                                                                                                                                                                                                                                                                        _v322 = _v321 - _v120;
                                                                                                                                                                                                                                                                                                        lhsZ[3][3][2][k][i][j] = _v322;
                                                                                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                                                                                            double _v323, _v325, _v324, _v326, _v327;
                                                                                                                                                                                                                                                                                                            _v323 = fjacZ[3][4][_v223][i][j];
                                                                                                                                                                                                                                                                                                            _v325 = njacZ[3][4][_v223][i][j];
                                                                                                                                                                                                                                                                                                            _v324 = _v4 * _v323;
                                                                                                                                                                                                                                                                                                            _v326 = _v2 * _v325;
                                                                                                                                                                                                                                                                                                            _v327 = _v324 - _v326;
                                                                                                                                                                                                                                                                                                            lhsZ[3][4][2][k][i][j] = _v327;
                                                                                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                                                                                double _v328, _v330, _v329, _v331, _v332;
                                                                                                                                                                                                                                                                                                                _v328 = fjacZ[4][0][_v223][i][j];
                                                                                                                                                                                                                                                                                                                _v330 = njacZ[4][0][_v223][i][j];
                                                                                                                                                                                                                                                                                                                _v329 = _v4 * _v328;
                                                                                                                                                                                                                                                                                                                _v331 = _v2 * _v330;
                                                                                                                                                                                                                                                                                                                _v332 = _v329 - _v331;
                                                                                                                                                                                                                                                                                                                lhsZ[4][0][2][k][i][j] = _v332;
                                                                                                                                                                                                                                                                                                                {
                                                                                                                                                                                                                                                                                                                    double _v333, _v335, _v334, _v336, _v337;
                                                                                                                                                                                                                                                                                                                    _v333 = fjacZ[4][1][_v223][i][j];
                                                                                                                                                                                                                                                                                                                    _v335 = njacZ[4][1][_v223][i][j];
                                                                                                                                                                                                                                                                                                                    _v334 = _v4 * _v333;
                                                                                                                                                                                                                                                                                                                    _v336 = _v2 * _v335;
                                                                                                                                                                                                                                                                                                                    _v337 = _v334 - _v336;
                                                                                                                                                                                                                                                                                                                    lhsZ[4][1][2][k][i][j] = _v337;
                                                                                                                                                                                                                                                                                                                    {
                                                                                                                                                                                                                                                                                                                        double _v338, _v340, _v339, _v341, _v342;
                                                                                                                                                                                                                                                                                                                        _v338 = fjacZ[4][2][_v223][i][j];
                                                                                                                                                                                                                                                                                                                        _v340 = njacZ[4][2][_v223][i][j];
                                                                                                                                                                                                                                                                                                                        _v339 = _v4 * _v338;
                                                                                                                                                                                                                                                                                                                        _v341 = _v2 * _v340;
                                                                                                                                                                                                                                                                                                                        _v342 = _v339 - _v341;
                                                                                                                                                                                                                                                                                                                        lhsZ[4][2][2][k][i][j] = _v342;
                                                                                                                                                                                                                                                                                                                        {
                                                                                                                                                                                                                                                                                                                            double _v343, _v345, _v344, _v346, _v347;
                                                                                                                                                                                                                                                                                                                            _v343 = fjacZ[4][3][_v223][i][j];
                                                                                                                                                                                                                                                                                                                            _v345 = njacZ[4][3][_v223][i][j];
                                                                                                                                                                                                                                                                                                                            _v344 = _v4 * _v343;
                                                                                                                                                                                                                                                                                                                            _v346 = _v2 * _v345;
                                                                                                                                                                                                                                                                                                                            _v347 = _v344 - _v346;
                                                                                                                                                                                                                                                                                                                            lhsZ[4][3][2][k][i][j] = _v347;
                                                                                                                                                                                                                                                                                                                            {
                                                                                                                                                                                                                                                                                                                                double _v348, _v350, _v349, _v351, _v352, _v353;
                                                                                                                                                                                                                                                                                                                                _v348 = fjacZ[4][4][_v223][i][j];
                                                                                                                                                                                                                                                                                                                                _v350 = njacZ[4][4][_v223][i][j];
                                                                                                                                                                                                                                                                                                                                _v349 = _v4 * _v348;
                                                                                                                                                                                                                                                                                                                                _v351 = _v2 * _v350;
                                                                                                                                                                                                                                                                                                                                _v352 = _v349 - _v351;
                                                                                                                                                                                                                                                                                                                                _v353 = _v352 - _v153;
                                                                                                                                                                                                                                                                                                                                lhsZ[4][4][2][k][i][j] = _v353;
                                                                                                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                                                                                                }
                                                                                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                                                                                }
                                                                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                                                                }
                                                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                                                }
                                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                                }
                                                                                                                                                                                                                                            }
                                                                                                                                                                                                                                        }
                                                                                                                                                                                                                                    }
                                                                                                                                                                                                                                }
                                                                                                                                                                                                                            }
                                                                                                                                                                                                                        }
                                                                                                                                                                                                                    }
                                                                                                                                                                                                                }
                                                                                                                                                                                                            }
                                                                                                                                                                                                        }
                                                                                                                                                                                                    }
                                                                                                                                                                                                }
                                                                                                                                                                                            }
                                                                                                                                                                                        }
                                                                                                                                                                                    }
                                                                                                                                                                                }
                                                                                                                                                                            }
                                                                                                                                                                        }
                                                                                                                                                                    }
                                                                                                                                                                }
                                                                                                                                                            }
                                                                                                                                                        }
                                                                                                                                                    }
                                                                                                                                                }
                                                                                                                                            }
                                                                                                                                        }
                                                                                                                                    }
                                                                                                                                }
                                                                                                                            }
                                                                                                                        }
                                                                                                                    }
                                                                                                                }
                                                                                                            }
                                                                                                        }
                                                                                                    }
                                                                                                }
                                                                                            }
                                                                                        }
                                                                                    }
                                                                                }
                                                                            }
                                                                        }
                                                                    }
                                                                }
                                                            }
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
    }
}
